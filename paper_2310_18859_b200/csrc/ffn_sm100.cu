// Expert FFN as a grouped bf16 GEMM on the 5th-gen tensor cores (sm_100a):
// TMA-fed, tcgen05.mma with the accumulator in TMEM, warp-specialised,
// persistent, with the bias/ReLU (GEMM1) and bias/alpha/unpermute/residual
// (GEMM2) epilogues fused. Replaces ref moe.py:235-262 (moe_apply), whose
// per-token gathered einsum is the reference's dominant cost.
//
// One launch = one GEMM over every (expert, row tile, BN-col tile) of a layer.
// Rows are the permuted (token, rank) rows of sida_permute_hist, so each
// expert's rows are contiguous: tile (e, m) covers rows off[e] + TM*m ... The
// B operand (W1^T or W2^T) is addressed in the HBM slot arena through a 3-D
// tensor map (k, n, slot): the residency engine moves experts between slots
// without rebuilding descriptors.
//
// Two CTA-group modes (template CG):
//   CG=1  one CTA per 128-row tile (small per-expert row counts)
//   CG=2  a CTA pair (cluster of 2 on one TPC) per 256-row tile:
//         tcgen05.mma.cta_group::2 (M=256) issued by the leader CTA, each CTA
//         TMA-loading its own 128 rows of A and half of the B tile, so per SM
//         the smem fill per MMA is 2/3 of CG=1 and the L2 reads of B halve.
//
// CTA = 10 warps: warp 0    TMA producer (one elected lane)
//                 warp 1    TMEM allocator + MMA issuer (one lane, leader CTA)
//                 warps 2-9 epilogue, two per TMEM lane quarter (each half of
//                           the tile's columns): TMEM -> registers -> swizzled
//                           smem transpose -> coalesced global stores
// Pipelines: smem ring of {A,B} stages (full/empty mbarriers); double-buffered
// TMEM accumulator (tmem_full/tmem_empty) so the epilogue of tile i overlaps
// the MMAs of tile i+1.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace sida {
namespace sm100 {

constexpr int BM = 128;       // rows per CTA (one TMEM lane per row)
constexpr int BK = 64;        // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int UMMA_K = 16;    // K per tcgen05.mma for kind::f16
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quarter
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kMaxListed = 512;
constexpr int kMaxBf16K = 4;
constexpr int kSmemBudget = 222 * 1024;

// Per-warp epilogue staging tile: 32 rows x 32 columns of the output type.
template <int STAGE>
__host__ __device__ constexpr int stage_tile_bytes() { return 32 * 32 * (STAGE == 1 ? 2 : 4); }

template <int BN, int STAGE, int CG>
__host__ __device__ constexpr int stages_for() {
  return (kSmemBudget - 1024 - kEpiWarps * stage_tile_bytes<STAGE>() - 8 * 1024) /
                     (BM * BK * 2 + (BN / CG) * BK * 2) > 8
             ? 8
             : (kSmemBudget - 1024 - kEpiWarps * stage_tile_bytes<STAGE>() - 8 * 1024) /
                   (BM * BK * 2 + (BN / CG) * BK * 2);
}

__host__ __device__ constexpr uint32_t pow2_cols(uint32_t c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

struct GemmParams {
  int n_rows, kdim, ndim;
  const int32_t* off;          // K+1 expert row offsets (permuted order)
  int num_experts;
  const int32_t* expert_slot;  // expert -> slot
  const int32_t* expert_list;  // optional subset
  int n_list;
  const uint8_t* arena;
  size_t slot_stride;
  size_t bias_off;             // byte offset of this GEMM's bias inside a slot (bf16)
  uint16_t* hidden;            // GEMM1 output (n_rows, ndim) bf16
  const int32_t* row_map;      // GEMM2: output row of permuted row p
  const float* alpha;
  const float* resid;
  float* out;
  uint16_t* out_bf16;          // GEMM2: optional bf16 copy of out (next layer's GEMM input)
  const int32_t* bf16_map;     // optional: out_bf16 row of (out row t, rank r) = map[t*k + r]
  int bf16_k;                  // ranks per out row in bf16_map (1..kMaxBf16K)
  uint16_t* const* peer_bf16;  // optional: bf16 rows go to peer_bf16[v / peer_stride] row
  int peer_stride;             //   v % peer_stride (expert-parallel dispatch / return)
  int32_t* err_flag;
  unsigned long long* prof;    // optional per-CTA cycle counters (sida_debug_gemm_prof)
  int linear;                  // GEMM1 epilogue without the ReLU (sida_linear_bf16)
  // CTA-pair launches: an expert's last tile holding <= 128 rows runs as an
  // M=128 pair MMA (64 rows per CTA) at half the tensor time of M=256
  int half_tiles;
};

// prof slots per CTA: producer wait(empty), MMA wait(tmem_empty), MMA wait(full),
// MMA loop total, epilogue wait(tmem_full), epilogue loop total, tiles
constexpr int kProfSlots = 12;  // + [8] entry, [9] after the PDL wait, [10] exit (%globaltimer ns)
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long clk() { return clock64(); }

// PTX shims: sm100_ptx.cuh

// ------------------------------------------------------------ tile schedule
struct TileInfo {
  int expert, row0, row_end, ncol0, slot;
  bool half;  // M=128 pair tile (see GemmParams::half_tiles)
};

// Destination of bf16 output row v: local out_bf16, or a (peer rank, row)
// pair encoded as rank * peer_stride + row into the peers' buffers.
__device__ __forceinline__ uint16_t* bf16_row(const GemmParams& p, int v) {
  if (p.peer_bf16) {
    const int q = v / p.peer_stride;
    return p.peer_bf16[q] + static_cast<size_t>(v - q * p.peer_stride) * p.ndim;
  }
  return p.out_bf16 + static_cast<size_t>(v) * p.ndim;
}

// First row of expert e (off == nullptr: one dense "expert" over all rows).
__device__ __forceinline__ int expert_row(const GemmParams& p, int e) {
  return p.off ? p.off[e] : (e == 0 ? 0 : p.n_rows);
}

// m-tile mt, column tile nt -> (expert, first row of the TM-row tile, ...).
__device__ __forceinline__ TileInfo decode_mt(int mt, int nt, const int32_t* s_prefix,
                                              const int32_t* s_expert, int n_list,
                                              const GemmParams& p, int BN, int TM) {
  int lo = 0, hi = n_list - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (s_prefix[mid] <= mt) lo = mid; else hi = mid - 1;
  }
  TileInfo ti;
  ti.expert = s_expert[lo];
  const int seg0 = expert_row(p, ti.expert);
  ti.row0 = seg0 + (mt - s_prefix[lo]) * TM;
  ti.row_end = expert_row(p, ti.expert + 1);
  ti.ncol0 = nt * BN;
  ti.slot = p.expert_slot ? p.expert_slot[ti.expert] : 0;
  ti.half = p.half_tiles && TM == 2 * BM && BN % 128 == 0 && ti.row_end - ti.row0 <= BM;
  return ti;
}

// Tile t -> (expert, first row of the TM-row tile, column tile).
__device__ __forceinline__ TileInfo decode_tile(int t, int n_ntiles, const int32_t* s_prefix,
                                                const int32_t* s_expert, int n_list,
                                                const GemmParams& p, int BN, int TM) {
  const int mt = t / n_ntiles;
  return decode_mt(mt, t - mt * n_ntiles, s_prefix, s_expert, n_list, p, BN, TM);
}

template <int BN, int STAGE, int CG>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmParams p) {
  // STAGE 1: GEMM1 (bias+ReLU -> hidden), 2: GEMM2 (alpha, unpermute, residual)
  constexpr int TM = BM * CG;                    // rows per tile (per CTA pair)
  constexpr int BNL = BN / CG;                   // B rows this CTA loads
  constexpr uint32_t kABytes = BM * BK * 2;
  constexpr uint32_t kBBytes = BNL * BK * 2;
  constexpr uint32_t kTmemCols = pow2_cols(2 * BN);
  constexpr int kStages = stages_for<BN, STAGE, CG>();
  constexpr int kTile = stage_tile_bytes<STAGE>();

  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for SWIZZLE_128B, as an offset from the shared array so
  // every derived pointer keeps the shared address space (LDS/STS, not LD.E/ST.E)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint8_t* sOut = sB + kStages * kBBytes;  // kEpiWarps staging tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + kEpiWarps * kTile);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tmem_full = bars + 2 * kStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  int32_t* s_prefix = reinterpret_cast<int32_t*>(s_tmem + 4);
  int32_t* s_expert = s_prefix + kMaxListed + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_list = p.expert_list ? p.n_list : p.num_experts;
  const uint32_t rank = CG == 1 ? 0u : cluster_rank();
  const bool leader = rank == 0;
  const int unit = blockIdx.x / CG, n_units = gridDim.x / CG;  // CTA pairs walk tiles together
  if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * kProfSlots + 8] = gtime();

  if (warp == 2) {
    // m-tile prefix over the listed experts: one warp, 32 experts per step
    // (a serial loop here costs one dependent L2 round trip per expert,
    // ~35 us at 128 experts, exposed because two of these CTAs cannot share
    // an SM, so the prologue cannot overlap the previous launch's tail)
    int acc = 0;
    for (int i0 = 0; i0 < n_list; i0 += 32) {
      const int i = i0 + lane;
      int cnt = 0, e = 0;
      if (i < n_list) {
        e = p.expert_list ? p.expert_list[i] : i;
        cnt = ceil_div(expert_row(p, e + 1) - expert_row(p, e), TM);
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (i < n_list) {
        s_expert[i] = e;
        s_prefix[i] = acc + incl - cnt;
      }
      acc += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_prefix[n_list] = acc;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], CG * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(s_tmem)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(s_tmem)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (CG == 1) __syncthreads(); else cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;
  // programmatic dependent launch: everything above (barriers, TMEM, tile
  // table) overlapped the previous kernel's tail; its outputs (A rows,
  // residual) are read only after it has completed and flushed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * kProfSlots + 9] = gtime();

  const int n_ntiles = p.ndim / BN;
  const int MT = s_prefix[n_list];
  const int total = MT * n_ntiles;
  auto item_subs = [&](int) -> int { return 1; };
  // work item -> (GEMM2?, m-tile, tile info)
  auto get_tile = [&](int it, int, bool& g2, int& mt) -> TileInfo {
    g2 = STAGE == 2;
    mt = it / n_ntiles;
    return decode_mt(mt, it - mt * n_ntiles, s_prefix, s_expert, n_list, p, BN, TM);
  };

  if (warp == 0) {
    // ===== TMA producer (both CTAs): own 128 rows of A, own BN/CG rows of B;
    // the warp walks the schedule in lockstep, one elected lane issues
    {
      int stage = 0;
      uint32_t phase = 0;
      unsigned long long w_empty = 0;
      for (int it = unit; it < total; it += n_units) {
      const int nsub = item_subs(it);
      for (int j = 0; j < nsub; ++j) {
        bool g2;
        int mt;
        const TileInfo ti = get_tile(it, j, g2, mt);
        if (ti.slot < 0) continue;
        const CUtensorMap* ta = &tmA;
        const CUtensorMap* tb = &tmB;
        const int nkb = p.kdim / BK;
        for (int kb = 0; kb < nkb; ++kb) {
          const unsigned long long c0 = p.prof ? clk() : 0;
          mbar_wait(&empty[stage], phase ^ 1);
          if (p.prof) w_empty += clk() - c0;
          const uint32_t fb = CG == 1 ? smem_u32(&full[stage]) : map_rank(smem_u32(&full[stage]), 0);
          if (elect_one()) {
            if (leader) mbar_expect_tx(&full[stage], CG * (kABytes + kBBytes));
            // (an M=128 pair tile takes rows [64 r, 64 r + 64) of CTA r: the
            // first half of its 128-row box)
            tma_load_2d<CG>(sA + stage * kABytes, ta, kb * BK,
                            ti.row0 + rank * (ti.half ? BM / 2 : BM), fb);
            tma_load_3d<CG>(sB + stage * kBBytes, tb, kb * BK, ti.ncol0 + rank * BNL, ti.slot, fb);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
      }
      if (p.prof && lane == 0) p.prof[blockIdx.x * kProfSlots + 0] = w_empty;
    }
  } else if (warp == 1) {
    // ===== MMA issuer: the whole warp walks the schedule in lockstep (the
    // descriptors stay warp-uniform, in uniform registers), one elected lane
    // issues the MMAs and the commits (leader CTA)
    if (leader) {
      constexpr uint32_t idesc_full = idesc_bf16<TM, BN>();
      constexpr uint32_t idesc_half = idesc_bf16<(TM > BM ? TM / 2 : TM), BN>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      unsigned long long w_epi = 0, w_tma = 0, n_tiles = 0;
      const unsigned long long m0 = p.prof ? clk() : 0;
      for (int it = unit; it < total; it += n_units) {
      const int nsub = item_subs(it);
      for (int j = 0; j < nsub; ++j) {
        bool g2;
        int mt;
        const TileInfo ti = get_tile(it, j, g2, mt);
        if (ti.slot < 0) {
          if (lane == 0) atomicExch(p.err_flag, 1);
          continue;
        }
        const int n_kblocks = p.kdim / BK;
        const uint32_t idesc = ti.half ? idesc_half : idesc_full;
        ++n_tiles;
        const unsigned long long c0 = p.prof ? clk() : 0;
        if constexpr (CG == 1) mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        else mbar_wait_cluster(&tmem_empty[acc], acc_phase ^ 1);
        if (p.prof) w_epi += clk() - c0;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * (kTmemCols / 2);
        for (int kb = 0; kb < n_kblocks; ++kb) {
          const unsigned long long c1 = p.prof ? clk() : 0;
          mbar_wait(&full[stage], phase);
          if (p.prof) w_tma += clk() - c1;
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * kABytes);
          const uint32_t b0 = smem_u32(sB + stage * kBBytes);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              umma_bf16<CG>(d_tmem, sw128_desc(a0 + k * UMMA_K * 2),
                            sw128_desc(b0 + k * UMMA_K * 2), idesc, (kb | k) != 0);
            }
            tc_commit<CG>(&empty[stage]);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) tc_commit<CG>(&tmem_full[acc]);
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      }
      if (p.prof && lane == 0) {
        unsigned long long* pr = p.prof + blockIdx.x * kProfSlots;
        pr[1] = w_epi;
        pr[2] = w_tma;
        pr[3] = clk() - m0;
        pr[6] = n_tiles;
      }
    }
  } else {
    // ===== epilogue. Warp w owns TMEM lanes 32*(w%4)..+31 (this CTA's tile
    // rows) and one half of the columns, in 32-column chunks. Per chunk:
    // tcgen05.ld (next chunk's load in flight), + bias, activation / alpha,
    // write the 32x32 sub-tile row-per-lane into a swizzled smem tile, then
    // re-read it column-chunk-per-lane so each global access covers whole row
    // segments (GEMM1: 8 rows x 64 B, GEMM2: 4 rows x 128 B per instruction).
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int kHalfCols = BN / 2;
    constexpr int kChunks = kHalfCols / 32;
    const uint32_t stile = smem_u32(sOut + (warp - 2) * kTile);
    int acc = 0;
    uint32_t acc_phase = 0;
    unsigned long long w_full = 0;
    const unsigned long long e0 = p.prof ? clk() : 0;
    for (int it = unit; it < total; it += n_units) {
      const int nsub = item_subs(it);
      for (int j = 0; j < nsub; ++j) {
      bool g2;
      int mt;
      const TileInfo ti = get_tile(it, j, g2, mt);
      if (ti.slot < 0) continue;
      const bool st2 = STAGE == 2;
      const GemmParams& gp = p;
      // first row of this warp's quarter. An M=128 pair tile's accumulator
      // (64 rows per CTA) sits in TMEM as two halves: N columns [0, BN/2) in
      // lanes 0-63 and [BN/2, BN) in lanes 64-127, each over BN/2 columns
      const int qrow0 = ti.half ? ti.row0 + rank * (BM / 2) + (quarter & 1) * 32
                                : ti.row0 + rank * BM + quarter * 32;
      const int my_row = qrow0 + lane;
      const bool valid = my_row < ti.row_end;
      const uint16_t* bias = reinterpret_cast<const uint16_t*>(
          gp.arena + static_cast<size_t>(ti.slot) * gp.slot_stride + gp.bias_off);
      float a_scale = 1.f;
      int orow = my_row;
      int brow[kMaxBf16K] = {};
      if (st2 && valid) {
        if (gp.alpha) a_scale = gp.alpha[my_row];
        if (gp.row_map) orow = gp.row_map[my_row];
        if (gp.bf16_map) {
#pragma unroll
          for (int r = 0; r < kMaxBf16K; ++r)
            if (r < gp.bf16_k) brow[r] = gp.bf16_map[static_cast<size_t>(orow) * gp.bf16_k + r];
        }
      }
      const int cbase = ti.half ? ti.ncol0 + (quarter >> 1) * kHalfCols + half * (kHalfCols / 2)
                                : ti.ncol0 + half * kHalfCols;
      const int nchunks = ti.half ? kChunks / 2 : kChunks;
      // GEMM2 residual rows, one chunk ahead: chunk c + 1's loads are in
      // flight while chunk c is stored (chunk 0's while the MMAs finish), so
      // the epilogue keeps two chunks of residual reads outstanding
      float4 xa[8], xb[8];
      auto load_x = [&](int c, float4 (&x)[8]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + (lane >> 3), q = lane & 7;
          const int orow_r = __shfl_sync(0xffffffffu, orow, r);
          x[i] = (gp.resid && qrow0 + r < ti.row_end)
                     ? __ldg(reinterpret_cast<const float4*>(
                           gp.resid + static_cast<size_t>(orow_r) * gp.ndim + cbase + c * 32 + q * 4))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      // (BN = 256: four chunks per warp leave no registers for a second
      // chunk of residual, so it loads each chunk at the chunk's start)
      constexpr bool kAhead = BN <= 192;
      if (st2 && kAhead) load_x(0, xa);
      const unsigned long long c2 = p.prof ? clk() : 0;
      mbar_wait(&tmem_full[acc], acc_phase);
      if (p.prof) w_full += clk() - c2;
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                             acc * (kTmemCols / 2) + half * (ti.half ? kHalfCols / 2 : kHalfCols);
      uint32_t v[2][32];
      tmem_ld32_nowait(t_row, v[0]);
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        if (kChunks % 2 == 0 && c == kChunks / 2 && nchunks == kChunks / 2) break;
        if (st2 && kAhead && c + 1 < nchunks) load_x(c + 1, (c & 1) ? xa : xb);
        if (st2 && !kAhead) load_x(c, (c & 1) ? xb : xa);
        const int col0 = cbase + c * 32;
        const uint4* bvec = reinterpret_cast<const uint4*>(bias + col0);
        uint4 braw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) braw[q] = __ldg(bvec + q);
        tmem_wait_ld();
        if (c + 1 < nchunks) tmem_ld32_nowait(t_row + (c + 1) * 32, v[(c + 1) & 1]);
        const uint32_t* vv = v[c & 1];
        float f[32];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t w[4] = {braw[q].x, braw[q].y, braw[q].z, braw[q].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            f[q * 8 + 2 * j] = __uint_as_float(vv[q * 8 + 2 * j]) + __uint_as_float(w[j] << 16);
            f[q * 8 + 2 * j + 1] =
                __uint_as_float(vv[q * 8 + 2 * j + 1]) + __uint_as_float(w[j] & 0xFFFF0000u);
          }
        }
        if (!st2) {
          // row-per-lane write: row r = lane, 4 x 16 B chunks, chunk' = q ^ ((r>>1)&3)
          const uint32_t srow = stile + lane * 64;
          const int sw = (lane >> 1) & 3;
#pragma unroll
          const float lo = gp.linear ? -INFINITY : 0.f;  // ReLU floor (none: linear)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 o;
            o.x = bf16x2_rn(fmaxf(f[q * 8 + 0], lo), fmaxf(f[q * 8 + 1], lo));
            o.y = bf16x2_rn(fmaxf(f[q * 8 + 2], lo), fmaxf(f[q * 8 + 3], lo));
            o.z = bf16x2_rn(fmaxf(f[q * 8 + 4], lo), fmaxf(f[q * 8 + 5], lo));
            o.w = bf16x2_rn(fmaxf(f[q * 8 + 6], lo), fmaxf(f[q * 8 + 7], lo));
            sts128(srow + ((q ^ sw) << 4), o);
          }
          __syncwarp();
          // read back: lane -> (row = i*8 + lane/4, chunk = lane%4)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = i * 8 + (lane >> 2), q = lane & 3;
            const uint4 val = lds128(stile + r * 64 + ((q ^ ((r >> 1) & 3)) << 4));
            if (qrow0 + r < ti.row_end)
              *reinterpret_cast<uint4*>(gp.hidden + static_cast<size_t>(qrow0 + r) * gp.ndim +
                                        col0 + q * 8) = val;
          }
          __syncwarp();
        } else {
          // row-per-lane write of alpha*(acc+b2): 8 x 16 B chunks, chunk' = q ^ (r & 7)
          const uint32_t srow = stile + lane * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4 o = make_float4(f[q * 4 + 0] * a_scale, f[q * 4 + 1] * a_scale,
                                   f[q * 4 + 2] * a_scale, f[q * 4 + 3] * a_scale);
            sts128(srow + ((q ^ (lane & 7)) << 4), *reinterpret_cast<uint4*>(&o));
          }
          __syncwarp();
          // read back: lane -> (row = i*4 + lane/8, chunk = lane%8); residual
          // (loaded one chunk ahead, load_x) and unpermute (row_map) per row segment
          const float4 (&x8)[8] = (c & 1) ? xb : xa;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + (lane >> 3), q = lane & 7;
            const int orow_r = __shfl_sync(0xffffffffu, orow, r);
            int brow8[kMaxBf16K];
            if (gp.bf16_map) {
#pragma unroll
              for (int j = 0; j < kMaxBf16K; ++j) brow8[j] = __shfl_sync(0xffffffffu, brow[j], r);
            }
            const uint4 raw = lds128(stile + r * 128 + ((q ^ (r & 7)) << 4));
            if (qrow0 + r < ti.row_end) {
              float4 o = *reinterpret_cast<const float4*>(&raw);
              const size_t at = static_cast<size_t>(orow_r) * gp.ndim + col0 + q * 4;
              if (gp.resid) {
                const float4 x = x8[i];
                o.x = x.x + o.x; o.y = x.y + o.y; o.z = x.z + o.z; o.w = x.w + o.w;
              }
              if (gp.out) *reinterpret_cast<float4*>(gp.out + at) = o;
              if (gp.out_bf16 || gp.peer_bf16) {
                uint2 ob;
                ob.x = bf16x2_rn(o.x, o.y);
                ob.y = bf16x2_rn(o.z, o.w);
                const int col = col0 + (lane & 7) * 4;
                if (!gp.bf16_map) {
                  if (!gp.peer_bf16)
                    *reinterpret_cast<uint2*>(gp.out_bf16 + at) = ob;
                  else
                    *reinterpret_cast<uint2*>(
                        bf16_row(gp, orow_r) + col) = ob;
                } else {  // expert-sorted copies: one per rank of this token
#pragma unroll
                  for (int j = 0; j < kMaxBf16K; ++j)
                    if (j < gp.bf16_k)
                      *reinterpret_cast<uint2*>(bf16_row(gp, brow8[j]) + col) = ob;
                }
              }
            }
          }
          __syncwarp();
        }
      }
      // this warp's TMEM reads are done: release the accumulator (leader's barrier)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        const uint32_t eb = smem_u32(&tmem_empty[acc]);
        mbar_arrive_cluster(CG == 1 ? eb : map_rank(eb, 0));
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
      }
    if (p.prof && warp == 2 && lane == 0) {
      p.prof[blockIdx.x * kProfSlots + 4] = w_full;
      p.prof[blockIdx.x * kProfSlots + 5] = clk() - e0;
    }
  }

  tc_fence_before();
  if constexpr (CG == 1) __syncthreads(); else cluster_sync();
  if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * kProfSlots + 10] = gtime();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(kTmemCols));
  }
}

// ------------------------------------------------------------ token-N tiles
// Swap-AB variant for experts holding few rows (many-expert layers): the
// expert's weight rows are the UMMA M side (256 output features per CTA pair,
// cta_group::2) and its token rows the N side, sized per expert in steps of 16
// (tcgen05 cost is proportional to N), so an expert of R rows wastes at most
// 15 rows per tile instead of up to 127 (BM = 128 token tiles: 2.5 tiles of
// MMA for 2 tiles of work at 256 rows per expert). D in TMEM is
// (feature lane, token column): each epilogue thread owns one output feature
// and walks 32 tokens per tcgen05.ld, so for a fixed token a warp's stores
// cover 32 consecutive features (64 B bf16 / 128 B fp32 row segments) and
// need no shared-memory transpose.
constexpr int kTnMax = 256;     // tokens per tile (UMMA N, pair)
constexpr int kTnBox = 64;      // token rows per TMA box
constexpr int kTnStages = 6;    // {A 16 KB, B <= 16 KB} per CTA

// Token tiles of an expert with R rows: count tiles of `base` rows (multiple
// of 16, <= 256), balanced so the last tile is not a sliver.
__device__ __forceinline__ void tn_split(int R, int& base, int& count) {
  if (R <= 0) { base = 16; count = 0; return; }
  const int n = ceil_div(R, kTnMax);
  base = min(kTnMax, (ceil_div(R, n) + 15) & ~15);
  count = ceil_div(R, base);
}

__device__ __forceinline__ uint32_t idesc_bf16_rt(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

struct TnTile {
  int expert, row0, nrows, nmma, f0, slot;
};

template <int STAGE>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_tn_kernel(const __grid_constant__ CUtensorMap tmW,  // (k, feature, slot), box 64x128
                       const __grid_constant__ CUtensorMap tmX,  // (k, row), box 64x32
                       const GemmParams p) {
  // STAGE 1: hidden = relu(X W1^T + b1); STAGE 2: out = alpha (H W2^T + b2) + resid
  constexpr uint32_t kABytes = 128 * BK * 2;
  constexpr uint32_t kBBytes = (kTnMax / 2) * BK * 2;
  constexpr uint32_t kBoxBytes = kTnBox * BK * 2;
  constexpr uint32_t kTmemCols = 2 * kTnMax;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kTnStages * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kTnStages * kBBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kTnStages;
  uint64_t* tmem_full = bars + 2 * kTnStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  int32_t* s_prefix = reinterpret_cast<int32_t*>(s_tmem + 4);
  int32_t* s_expert = s_prefix + kMaxListed + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_list = p.expert_list ? p.n_list : p.num_experts;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int unit = blockIdx.x >> 1, n_units = gridDim.x >> 1;
  if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * kProfSlots + 8] = gtime();

  if (warp == 2) {
    // token-tile prefix over the listed experts: one warp, 32 experts per step
    int acc = 0;
    for (int i0 = 0; i0 < n_list; i0 += 32) {
      const int i = i0 + lane;
      int cnt = 0, e = 0;
      if (i < n_list) {
        e = p.expert_list ? p.expert_list[i] : i;
        int base;
        tn_split(expert_row(p, e + 1) - expert_row(p, e), base, cnt);
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (i < n_list) {
        s_expert[i] = e;
        s_prefix[i] = acc + incl - cnt;
      }
      acc += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_prefix[n_list] = acc;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTnStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * kProfSlots + 9] = gtime();

  const int n_ft = p.ndim / 256;  // feature tiles per expert (M = 256 per pair)
  const int total = s_prefix[n_list] * n_ft;
  const int nkb = p.kdim / BK;
  auto get_tile = [&](int it) -> TnTile {
    const int mt = it / n_ft;
    const int nt = it - mt * n_ft;
    int lo = 0, hi = n_list - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_prefix[mid] <= mt) lo = mid; else hi = mid - 1;
    }
    TnTile t;
    t.expert = s_expert[lo];
    const int seg0 = expert_row(p, t.expert);
    const int R = expert_row(p, t.expert + 1) - seg0;
    int base, cnt;
    tn_split(R, base, cnt);
    const int j = mt - s_prefix[lo];
    t.row0 = seg0 + j * base;
    t.nrows = min(base, R - j * base);
    t.nmma = (t.nrows + 15) & ~15;
    t.f0 = nt * 256;
    t.slot = p.expert_slot ? p.expert_slot[t.expert] : 0;
    return t;
  };

  if (warp == 0) {
    // ===== TMA producer (both CTAs): own 128 weight rows, own half of the
    // tokens (warp-uniform walk, one elected lane issues)
    {
      int stage = 0;
      uint32_t phase = 0;
      unsigned long long w_empty = 0;
      for (int it = unit; it < total; it += n_units) {
        const TnTile t = get_tile(it);
        if (t.slot < 0) continue;
        const int half_rows = t.nmma >> 1;
        const int nbox = ceil_div(half_rows, kTnBox);
        const int xrow = t.row0 + static_cast<int>(rank) * half_rows;
        for (int kb = 0; kb < nkb; ++kb) {
          const unsigned long long c0 = p.prof ? clk() : 0;
          mbar_wait(&empty[stage], phase ^ 1);
          if (p.prof) w_empty += clk() - c0;
          const uint32_t fb = map_rank(smem_u32(&full[stage]), 0);
          if (elect_one()) {
            if (leader) mbar_expect_tx(&full[stage], 2 * (kABytes + nbox * kBoxBytes));
            tma_load_3d<2>(sA + stage * kABytes, &tmW, kb * BK, t.f0 + rank * 128, t.slot, fb);
            for (int b = 0; b < nbox; ++b)
              tma_load_2d<2>(sB + stage * kBBytes + b * kBoxBytes, &tmX, kb * BK,
                             xrow + b * kTnBox, fb);
          }
          __syncwarp();
          if (++stage == kTnStages) { stage = 0; phase ^= 1; }
        }
      }
      if (p.prof && lane == 0) p.prof[blockIdx.x * kProfSlots + 0] = w_empty;
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA): M = 256 features x N = nmma tokens;
    // warp-uniform walk, one elected lane issues
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const unsigned long long m0 = p.prof ? clk() : 0;
      unsigned long long w_epi = 0, w_tma = 0, n_tiles = 0;
      for (int it = unit; it < total; it += n_units) {
        const TnTile t = get_tile(it);
        if (t.slot < 0) {
          if (lane == 0) atomicExch(p.err_flag, 1);
          continue;
        }
        const uint32_t idesc = idesc_bf16_rt(256, t.nmma);
        ++n_tiles;
        const unsigned long long c1 = p.prof ? clk() : 0;
        mbar_wait_cluster(&tmem_empty[acc], acc_phase ^ 1);
        if (p.prof) w_epi += clk() - c1;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kTnMax;
        for (int kb = 0; kb < nkb; ++kb) {
          const unsigned long long c2 = p.prof ? clk() : 0;
          mbar_wait(&full[stage], phase);
          if (p.prof) w_tma += clk() - c2;
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * kABytes);
          const uint32_t b0 = smem_u32(sB + stage * kBBytes);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k)
              umma_bf16<2>(d_tmem, sw128_desc(a0 + k * UMMA_K * 2),
                           sw128_desc(b0 + k * UMMA_K * 2), idesc, (kb | k) != 0);
            tc_commit<2>(&empty[stage]);
          }
          __syncwarp();
          if (++stage == kTnStages) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) tc_commit<2>(&tmem_full[acc]);
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (p.prof && lane == 0) {
        unsigned long long* pr = p.prof + blockIdx.x * kProfSlots;
        pr[1] = w_epi;
        pr[2] = w_tma;
        pr[3] = clk() - m0;
        pr[6] = n_tiles;
      }
    }
  } else {
    // ===== epilogue: warp owns TMEM lanes 32*(w%4).. (32 features of this
    // CTA's 128) and every other 32-token chunk of the tile
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    const unsigned long long e0 = p.prof ? clk() : 0;
    unsigned long long w_full = 0;
    for (int it = unit; it < total; it += n_units) {
      const TnTile t = get_tile(it);
      if (t.slot < 0) continue;
      const int f = t.f0 + static_cast<int>(rank) * 128 + quarter * 32 + lane;
      const uint16_t* bias = reinterpret_cast<const uint16_t*>(
          p.arena + static_cast<size_t>(t.slot) * p.slot_stride + p.bias_off);
      const float b = bf16_to_f32(bias[f]);
      const int nch = ceil_div(t.nrows, 32);
      const unsigned long long c3 = p.prof ? clk() : 0;
      mbar_wait(&tmem_full[acc], acc_phase);
      if (p.prof) w_full += clk() - c3;
      tc_fence_after();
      const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * kTnMax;
      for (int c = half; c < nch; c += 2) {
        uint32_t v[32];
        tmem_ld32_nowait(t_lane + c * 32, v);
        const int tok0 = t.row0 + c * 32;
        const int cnt = min(32, t.nrows - c * 32);
        if (STAGE == 1) {
          tmem_wait_ld();
          // lane pairs (f, f+1) trade halves so each lane stores one bf16x2
          // word per token pair: even lanes the even tokens, odd lanes the odd
          // ones (a warp store covers two 64 B row segments)
          const bool odd = lane & 1;
          uint32_t* dst = reinterpret_cast<uint32_t*>(
              p.hidden + static_cast<size_t>(tok0 + (odd ? 1 : 0)) * p.ndim + (f & ~1));
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float y0 = fmaxf(__uint_as_float(v[j]) + b, 0.f);
            const float y1 = fmaxf(__uint_as_float(v[j + 1]) + b, 0.f);
            const float other = __shfl_xor_sync(0xffffffffu, odd ? y0 : y1, 1);
            const uint32_t w = odd ? bf16x2_rn(other, y1) : bf16x2_rn(y0, other);
            if (j + (odd ? 1 : 0) < cnt) dst[static_cast<size_t>(j) * (p.ndim >> 1)] = w;
          }
        } else {
          // per-token row map / alpha: lane j holds token tok0 + j's, broadcast by shuffles
          const int my_tok = tok0 + lane;
          int orow_l = my_tok;
          float a_l = 1.f;
          if (lane < cnt) {
            if (p.row_map) orow_l = p.row_map[my_tok];
            if (p.alpha) a_l = p.alpha[my_tok];
          }
          float x[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int o = __shfl_sync(0xffffffffu, orow_l, j);
            x[j] = (p.resid && j < cnt) ? __ldg(p.resid + static_cast<size_t>(o) * p.ndim + f) : 0.f;
          }
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int o = __shfl_sync(0xffffffffu, orow_l, j);
            const float a = __shfl_sync(0xffffffffu, a_l, j);
            if (j < cnt) {
              const float y = x[j] + (__uint_as_float(v[j]) + b) * a;
              const size_t at = static_cast<size_t>(o) * p.ndim + f;
              if (p.out) p.out[at] = y;
              if (p.out_bf16) p.out_bf16[at] = __bfloat16_as_ushort(__float2bfloat16_rn(y));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(map_rank(smem_u32(&tmem_empty[acc]), 0));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (p.prof && warp == 2 && lane == 0) {
      p.prof[blockIdx.x * kProfSlots + 4] = w_full;
      p.prof[blockIdx.x * kProfSlots + 5] = clk() - e0;
    }
  }

  tc_fence_before();
  cluster_sync();
  if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * kProfSlots + 10] = gtime();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

constexpr size_t tn_smem_bytes() {
  return 1024 + kTnStages * (128 * BK * 2 + (kTnMax / 2) * BK * 2) + (2 * kTnStages + 4) * 8 + 16 +
         (2 * kMaxListed + 2) * 4;
}

template <int BN, int STAGE, int CG>
constexpr size_t smem_bytes() {
  return 1024 + stages_for<BN, STAGE, CG>() * (BM * BK * 2 + (BN / CG) * BK * 2) +
         kEpiWarps * stage_tile_bytes<STAGE>() + (2 * stages_for<BN, STAGE, CG>() + 4) * 8 + 16 +
         (2 * kMaxListed + 2) * 4;
}

// ------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

static int make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                       uint32_t box_rows) {
  auto fn = encode_fn();
  SIDA_REQUIRE(fn, SIDA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SIDA_REQUIRE(r == CUDA_SUCCESS, SIDA_ERR_CUDA, "tensor map (2d) encode failed: %d", (int)r);
  return SIDA_OK;
}

static int make_map_3d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                       uint64_t slots, uint64_t slot_stride, uint32_t box_rows) {
  auto fn = encode_fn();
  SIDA_REQUIRE(fn, SIDA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {inner, rows, slots};
  cuuint64_t strides[2] = {inner * 2, slot_stride};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(BK), box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SIDA_REQUIRE(r == CUDA_SUCCESS, SIDA_ERR_CUDA, "tensor map (3d) encode failed: %d", (int)r);
  return SIDA_OK;
}

// Programmatic dependent launch of every grouped-GEMM launch (its prologue
// overlaps the previous kernel's tail); SIDA_PDL=0 turns it off (A/B).
static int pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SIDA_PDL");
    v = e ? atoi(e) : 1;
  }
  return v;
}

template <int BN, int STAGE, int CG>
static int launch_gemm(const void* a_base, const void* b_base, int n_slots, const GemmParams& p,
                       int n_listed, cudaStream_t s) {
  auto kern = grouped_gemm_kernel<BN, STAGE, CG>;
  static bool configured = false;
  if (!configured) {
    SIDA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_bytes<BN, STAGE, CG>()));
    configured = true;
  }
  CUtensorMap ta, tb;
  int st = make_map_2d(&ta, a_base, p.kdim, p.n_rows, BM);
  if (st) return st;
  st = make_map_3d(&tb, b_base, p.kdim, p.ndim, n_slots, p.slot_stride, BN / CG);
  if (st) return st;
  const int col_tiles = p.ndim / BN;
  const int max_tiles = (ceil_div(p.n_rows, BM * CG) + n_listed) * col_tiles;
  const int units = std::max(1, std::min(max_tiles, kNumSMs / CG));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units * CG);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes<BN, STAGE, CG>();
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  SIDA_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, p));
  count_launch();
  return SIDA_OK;
}

template <int STAGE, int CG>
static int dispatch_bn(const void* a_base, const void* b_base, int n_slots, const GemmParams& p,
                       int n_listed, cudaStream_t s) {
  // N tile: 256 whenever it divides N. The GEMMs are fed at close to the
  // L2->SM limit (~10 TB/s measured), so the widest tile (fewest A re-reads
  // per FLOP) wins even where a narrower one quantises better: d = 768 at
  // BN=256 reads the hidden rows 3x instead of 4x (0.312 -> 0.296 ms/layer).
  // SIDA_FFN_BN2=192|128 forces the GEMM2 tile for measurements.
  static int forced_bn = -1;
  if (forced_bn < 0) {
    const char* e = getenv("SIDA_FFN_BN2");
    forced_bn = e ? atoi(e) : 0;
  }
  if (STAGE == 2 && forced_bn == 192 && p.ndim % 192 == 0)
    return launch_gemm<192, STAGE, CG>(a_base, b_base, n_slots, p, n_listed, s);
  if (STAGE == 2 && forced_bn == 128 && p.ndim % 128 == 0)
    return launch_gemm<128, STAGE, CG>(a_base, b_base, n_slots, p, n_listed, s);
  if (p.ndim % 256 == 0)
    return launch_gemm<256, STAGE, CG>(a_base, b_base, n_slots, p, n_listed, s);
  if (p.ndim % 192 == 0) return launch_gemm<192, STAGE, CG>(a_base, b_base, n_slots, p, n_listed, s);
  if (p.ndim % 128 == 0) return launch_gemm<128, STAGE, CG>(a_base, b_base, n_slots, p, n_listed, s);
  return launch_gemm<64, STAGE, CG>(a_base, b_base, n_slots, p, n_listed, s);
}

// Token-N (swap-AB) launch: a_base = token rows (x_perm / hidden), b_base =
// the weight arena at this GEMM's matrix offset.
template <int STAGE>
static int launch_tn(const void* x_base, const void* w_base, int n_slots, const GemmParams& p,
                     int n_listed, cudaStream_t s) {
  auto kern = grouped_gemm_tn_kernel<STAGE>;
  static bool configured = false;
  if (!configured) {
    SIDA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)tn_smem_bytes()));
    configured = true;
  }
  CUtensorMap tw, tx;
  int st = make_map_3d(&tw, w_base, p.kdim, p.ndim, n_slots, p.slot_stride, 128);
  if (st) return st;
  if ((st = make_map_2d(&tx, x_base, p.kdim, p.n_rows, kTnBox))) return st;
  const int max_tiles = (ceil_div(p.n_rows, kTnMax) + n_listed) * (p.ndim / 256);
  const int units = std::max(1, std::min(max_tiles, kNumSMs / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units * 2);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = tn_smem_bytes();
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  SIDA_CUDA(cudaLaunchKernelEx(&cfg, kern, tw, tx, p));
  count_launch();
  return SIDA_OK;
}

// CTA-pair (M=256) tiles when experts hold enough rows to fill them.
template <int STAGE>
static int dispatch_gemm(const void* a_base, const void* b_base, int n_slots, const GemmParams& p,
                         int n_listed, int cg, cudaStream_t s) {
  if (cg == 2) return dispatch_bn<STAGE, 2>(a_base, b_base, n_slots, p, n_listed, s);
  return dispatch_bn<STAGE, 1>(a_base, b_base, n_slots, p, n_listed, s);
}

}  // namespace sm100
}  // namespace sida

using namespace sida;

static unsigned long long* g_prof = nullptr;  // [2 GEMMs][148 CTAs][kProfSlots]

static int g_prof_on = -1;  // SIDA_GEMM_PROF=1 at load, or sida_set_gemm_prof

static unsigned long long* prof_buffer(int gemm) {
  if (g_prof_on < 0) g_prof_on = getenv("SIDA_GEMM_PROF") != nullptr;
  if (!g_prof_on) return nullptr;
  if (!g_prof) {
    const size_t bytes = 2ull * kNumSMs * sm100::kProfSlots * sizeof(unsigned long long);
    if (cudaMalloc(&g_prof, bytes) != cudaSuccess) return nullptr;
    cudaMemset(g_prof, 0, bytes);
  }
  return g_prof + (size_t)gemm * kNumSMs * sm100::kProfSlots;
}

// Observability: turn the FFN GEMM profile counters on or off at run time.
extern "C" int sida_set_gemm_prof(int on) {
  g_prof_on = on ? 1 : 0;
  if (on) SIDA_REQUIRE(prof_buffer(0), SIDA_ERR_CUDA, "profile buffer allocation failed");
  return SIDA_OK;
}

// Observability: copy the per-CTA cycle counters of the last FFN call
// (enabled by SIDA_GEMM_PROF=1) into out[2][148][12]; synchronises the device.
extern "C" int sida_debug_gemm_prof(unsigned long long* out) {
  SIDA_REQUIRE(g_prof, SIDA_ERR_UNSUPPORTED, "run with SIDA_GEMM_PROF=1 to collect counters");
  SIDA_CUDA(cudaDeviceSynchronize());
  SIDA_CUDA(cudaMemcpy(out, g_prof, 2ull * kNumSMs * sm100::kProfSlots * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost));
  return SIDA_OK;
}

// CTA-group choice per GEMM: SIDA_FFN_CG=1|2 forces it; by default GEMM1
// (K = d: short k-loop) pairs up (M=256 tiles) once the average expert holds
// >= 1024 rows, GEMM2 (K = h) already at >= 192 rows: its pair tiles halve
// the weight re-reads, which outweighs their padding down to ~256 rows per
// expert (ncu, profiles/r1/ffn_tile_families.txt: base-128 GEMM2 197 vs
// 220 us, base-64 164 vs 177 us; at 128 rows both are equal).
static int choose_cg(int gemm, int n_rows, int listed) {
  static int forced = -1;
  if (forced < 0) {
    const char* e = getenv("SIDA_FFN_CG");
    forced = e ? atoi(e) : 0;
  }
  if (forced == 1 || forced == 2) return forced;
  (void)gemm;
  // pair tiles whenever experts average >= 96 rows: with the M=128 pair tile
  // for an expert's last <= 128 rows (half_tiles) they cost no more tensor
  // time than 128-row single-CTA tiles and stream each expert's weights to
  // the SMs fewer times (2.5 -> 1.5 per expert at 256 +- 16 rows)
  return n_rows >= 96 * listed ? 2 : 1;
}

// Tile family per expert GEMM (sida_set_ffn_tiles, or SIDA_FFN_SWAP at load):
// -1 auto, 0 token-M for both GEMMs, 1 token-N (swap-AB) for both, 2 token-M
// GEMM1 + token-N GEMM2, 3 token-N GEMM1 + token-M GEMM2, 5 the one-launch
// FFN of expert_ffn.cu (4, a per-token-tile fused kernel, was retired). Auto
// is token-N for both GEMMs wherever d, h % 256 == 0 -- measured fastest or
// equal at every expert count once the MMA issue is warp-uniform (one B200,
// tools/ffn_probe.py, 32K rows: base-128 0.400 vs 0.425 ms token-M, base-64
// 0.341 vs 0.352, base-256 0.530 vs 0.570, base-8 0.281 both; 131K rows at
// base-128 1.194 vs 1.211) -- and token-M with the CTA-group choice above
// otherwise. SIDA_FFN_SWAP sets the initial mode.
static int g_tn_mode = -2;

static void tn_init() {
  if (g_tn_mode != -2) return;
  const char* e = getenv("SIDA_FFN_SWAP");
  g_tn_mode = e ? atoi(e) : -1;
}

static bool choose_tn(int gemm, int d, int h) {
  tn_init();
  if (d % 256 != 0 || h % 256 != 0) return false;
  switch (g_tn_mode) {
    case 0: return false;
    case 2: return gemm == 2;
    case 3: return gemm == 1;
    default: return true;  // 1, and auto
  }
}

extern "C" int sida_set_ffn_tiles(int mode) {
  SIDA_REQUIRE(mode >= -1 && mode <= 5 && mode != 4, SIDA_ERR_CONTRACT,
               "ffn tile mode %d not in -1..3, 5 (4, the per-token-tile fused FFN, was retired)",
               mode);
  tn_init();
  g_tn_mode = mode;
  return SIDA_OK;
}

extern "C" int sida_get_ffn_tiles(void) {
  tn_init();
  return g_tn_mode;
}

// One persistent launch for both expert GEMMs (expert_ffn.cu): mode 5, or
// auto mode with SIDA_XFFN=1. Measured slower than the two token-M launches
// (tools/ffn_probe.py, one B200: base-8 0.389 vs 0.293 ms, base-128 0.464 vs
// 0.442 ms per layer), so auto keeps the two launches.
extern "C" int sida_expert_ffn_applicable(int d, int h);
extern "C" int sida_expert_ffn_launch(const uint16_t* x_perm, int n_rows, int d, int h,
                                      const int32_t* off, int num_experts,
                                      const int32_t* expert_slot, const int32_t* expert_list,
                                      int n_list, const void* arena, size_t slot_stride,
                                      int n_slots, const int32_t* row_map, const float* alpha,
                                      const float* resid, float* out, uint16_t* out_bf16,
                                      uint16_t* hidden, int32_t* err_flag, void* stream);

static bool choose_xffn(int d, int h) {
  tn_init();
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SIDA_XFFN");
    env = e ? atoi(e) : 0;
  }
  if (!sida_expert_ffn_applicable(d, h)) return false;
  return g_tn_mode == 5 || (g_tn_mode == -1 && env);
}

extern "C" int sida_grouped_ffn_bf16(const uint16_t* x_perm, int n_rows, int d, int h,
                                     const int32_t* off, int num_experts,
                                     const int32_t* expert_slot, const int32_t* expert_list,
                                     int n_list, const void* arena, size_t slot_stride,
                                     int n_slots, const int32_t* row_map, const float* alpha,
                                     const float* resid, float* out, uint16_t* out_bf16,
                                     uint16_t* hidden,
                                     int32_t* err_flag, void* stream) {
  SIDA_REQUIRE(d % 64 == 0 && h % 64 == 0, SIDA_ERR_UNSUPPORTED,
               "tcgen05 FFN needs d, h multiples of 64 (d=%d h=%d)", d, h);
  SIDA_REQUIRE(n_rows >= 0 && num_experts >= 1 && n_slots >= 1, SIDA_ERR_CONTRACT,
               "bad ffn dims rows=%d K=%d slots=%d", n_rows, num_experts, n_slots);
  const int listed = expert_list ? n_list : num_experts;
  SIDA_REQUIRE(listed <= sm100::kMaxListed, SIDA_ERR_UNSUPPORTED, "more than %d experts listed",
               sm100::kMaxListed);
  SIDA_REQUIRE(slot_stride % 16 == 0 && slot_stride >= sida_slot_bytes(d, h), SIDA_ERR_CONTRACT,
               "slot stride %zu invalid", slot_stride);
  SIDA_REQUIRE(err_flag && (out || out_bf16) && hidden && x_perm && off && expert_slot && arena,
               SIDA_ERR_CONTRACT, "null pointer passed to sida_grouped_ffn_bf16");
  if (n_rows == 0 || listed == 0) return SIDA_OK;
  cudaStream_t s = as_stream(stream);
  const uint8_t* ar = static_cast<const uint8_t*>(arena);
  const size_t w2_off = (size_t)h * d * 2, b1_off = 2 * w2_off, b2_off = b1_off + (size_t)h * 2;

  if (choose_xffn(d, h))
    return sida_expert_ffn_launch(x_perm, n_rows, d, h, off, num_experts, expert_slot,
                                  expert_list, n_list, arena, slot_stride, n_slots, row_map,
                                  alpha, resid, out, out_bf16, hidden, err_flag, stream);
  sm100::GemmParams p1{};
  p1.n_rows = n_rows; p1.kdim = d; p1.ndim = h;
  p1.off = off; p1.num_experts = num_experts; p1.expert_slot = expert_slot;
  p1.expert_list = expert_list; p1.n_list = n_list;
  p1.arena = ar; p1.slot_stride = slot_stride; p1.bias_off = b1_off;
  p1.hidden = hidden; p1.err_flag = err_flag; p1.prof = prof_buffer(0);
  p1.half_tiles = 1;
  int st = choose_tn(1, d, h) ? sm100::launch_tn<1>(x_perm, ar, n_slots, p1, listed, s)
              : sm100::dispatch_gemm<1>(x_perm, ar, n_slots, p1, listed,
                                        choose_cg(1, n_rows, listed), s);
  if (st) return st;

  sm100::GemmParams p2 = p1;
  p2.kdim = h; p2.ndim = d; p2.bias_off = b2_off;
  p2.row_map = row_map; p2.alpha = alpha; p2.resid = resid; p2.out = out;
  p2.out_bf16 = out_bf16;
  p2.prof = prof_buffer(1);
  if (choose_tn(2, d, h)) return sm100::launch_tn<2>(hidden, ar + w2_off, n_slots, p2, listed, s);
  return sm100::dispatch_gemm<2>(hidden, ar + w2_off, n_slots, p2, listed,
                                 choose_cg(2, n_rows, listed), s);
}

// Mixing-attention output projection with the residual and the next FFN's
// expert-sorted input fused into the epilogue (ref moe.py:232-233, then the
// row gather implicit in moe.py:253-256): out[t] = resid[t] + ctx[t] Wo and
// x_perm[inv[t*k + r]] = bf16(out[t]) for every rank r < k (k = 0: no copy).
// wo_t: Wo^T (d_out x d_in, bf16, K-major) followed by d_out zero bf16 (the
// bias slot of the grouped-GEMM epilogue), sida_out_proj_bytes(d) bytes.
extern "C" size_t sida_out_proj_bytes(int d) {
  return align_up(static_cast<size_t>(d) * d * 2 + static_cast<size_t>(d) * 2, 16);
}

extern "C" int sida_out_proj_scatter(const uint16_t* ctx, int n_rows, int d, const void* wo_t,
                                     const float* resid, float* out, const int32_t* inv, int k,
                                     uint16_t* x_perm, int32_t* err_flag, void* stream) {
  SIDA_REQUIRE(d % 64 == 0, SIDA_ERR_UNSUPPORTED, "out projection needs d multiple of 64 (d=%d)",
               d);
  SIDA_REQUIRE(n_rows >= 0 && k >= 0 && k <= sm100::kMaxBf16K, SIDA_ERR_CONTRACT,
               "bad out-projection dims rows=%d k=%d", n_rows, k);
  SIDA_REQUIRE(ctx && wo_t && resid && out && err_flag && (k == 0 || (inv && x_perm)),
               SIDA_ERR_CONTRACT, "null pointer passed to sida_out_proj_scatter");
  if (n_rows == 0) return SIDA_OK;
  sm100::GemmParams p{};
  p.n_rows = n_rows; p.kdim = d; p.ndim = d;
  p.off = nullptr; p.num_experts = 1; p.expert_slot = nullptr;
  p.arena = static_cast<const uint8_t*>(wo_t);
  p.slot_stride = sida_out_proj_bytes(d);
  p.bias_off = static_cast<size_t>(d) * d * 2;
  p.resid = resid; p.out = out;
  p.out_bf16 = k ? x_perm : nullptr; p.bf16_map = k ? inv : nullptr; p.bf16_k = k;
  p.err_flag = err_flag;
  const int cg = n_rows >= 1024 ? 2 : 1;
  // N tile 192 when it divides d: at d = 768 the 32K-row projection is 512
  // tiles (6.9 persistent rounds of 74 pairs) instead of 384 (5.2 rounds), and
  // this epilogue-bound GEMM gains more from the fuller last round than it
  // loses to the narrower tile (tools/proj_probe.py: 98 -> 92 us).
  // SIDA_OUTPROJ_BN=256|128 overrides (A/B).
  static int bn = -1;
  if (bn < 0) {
    const char* e = getenv("SIDA_OUTPROJ_BN");
    bn = e ? atoi(e) : 192;
  }
  if (bn == 192 && d % 192 == 0) {
    if (cg == 2) return sm100::launch_gemm<192, 2, 2>(ctx, wo_t, 1, p, 1, as_stream(stream));
    return sm100::launch_gemm<192, 2, 1>(ctx, wo_t, 1, p, 1, as_stream(stream));
  }
  if (bn == 128 && d % 128 == 0) {
    if (cg == 2) return sm100::launch_gemm<128, 2, 2>(ctx, wo_t, 1, p, 1, as_stream(stream));
    return sm100::launch_gemm<128, 2, 1>(ctx, wo_t, 1, p, 1, as_stream(stream));
  }
  return sm100::dispatch_gemm<2>(ctx, wo_t, 1, p, 1, cg, as_stream(stream));
}

// Dense bf16 linear layer on the same tcgen05 GEMM (one "expert" over every
// row, GEMM1 epilogue without the ReLU): out = x W (bf16), W given as
// w_t = W^T (n x k, bf16, K-major) followed by n bf16 bias values,
// sida_linear_bytes(k, n) bytes. The mixing attention's fused QKV projection
// (ref moe.py:225-227: q, k, v = x Wq, x Wk, x Wv as one n = 3d product).
extern "C" size_t sida_linear_bytes(int k, int n) {
  return align_up(static_cast<size_t>(n) * k * 2 + static_cast<size_t>(n) * 2, 16);
}

extern "C" int sida_linear_bf16(const uint16_t* x, int n_rows, int k, int n, const void* w_t,
                                uint16_t* out, int32_t* err_flag, void* stream) {
  SIDA_REQUIRE(k % 64 == 0 && n % 64 == 0, SIDA_ERR_UNSUPPORTED,
               "tcgen05 linear needs k, n multiples of 64 (k=%d n=%d)", k, n);
  SIDA_REQUIRE(n_rows >= 0, SIDA_ERR_CONTRACT, "bad linear rows=%d", n_rows);
  SIDA_REQUIRE(x && w_t && out && err_flag, SIDA_ERR_CONTRACT,
               "null pointer passed to sida_linear_bf16");
  if (n_rows == 0) return SIDA_OK;
  sm100::GemmParams p{};
  p.n_rows = n_rows; p.kdim = k; p.ndim = n;
  p.off = nullptr; p.num_experts = 1; p.expert_slot = nullptr;
  p.arena = static_cast<const uint8_t*>(w_t);
  p.slot_stride = sida_linear_bytes(k, n);
  p.bias_off = static_cast<size_t>(n) * k * 2;
  p.hidden = out; p.err_flag = err_flag; p.linear = 1;
  return sm100::dispatch_gemm<1>(x, w_t, 1, p, 1, n_rows >= 1024 ? 2 : 1, as_stream(stream));
}

// ---------------------------------------------------------------------------
// Expert parallelism over peer memory: the two data
// exchanges of an EP layer folded into the epilogues that produce the rows.
//
// Dispatch: the output projection writes each token's bf16 expert input
// straight into the OWNER rank's expert-major receive buffer: map[t*k + r] =
// owner * peer_stride + row, peers[q] = rank q's receive buffer (a peer /
// IPC mapping; over NVLink on a multi-GPU box).
extern "C" int sida_out_proj_scatter_peer(const uint16_t* ctx, int n_rows, int d,
                                          const void* wo_t, const float* resid, float* out,
                                          const int32_t* map, int k, uint16_t* const* peers,
                                          int peer_stride, int32_t* err_flag, void* stream) {
  SIDA_REQUIRE(d % 64 == 0, SIDA_ERR_UNSUPPORTED, "out projection needs d multiple of 64 (d=%d)",
               d);
  SIDA_REQUIRE(n_rows >= 0 && k >= 1 && k <= sm100::kMaxBf16K && peer_stride >= 1,
               SIDA_ERR_CONTRACT, "bad out-projection dims rows=%d k=%d", n_rows, k);
  SIDA_REQUIRE(ctx && wo_t && resid && out && err_flag && map && peers, SIDA_ERR_CONTRACT,
               "null pointer passed to sida_out_proj_scatter_peer");
  if (n_rows == 0) return SIDA_OK;
  sm100::GemmParams p{};
  p.n_rows = n_rows; p.kdim = d; p.ndim = d;
  p.off = nullptr; p.num_experts = 1; p.expert_slot = nullptr;
  p.arena = static_cast<const uint8_t*>(wo_t);
  p.slot_stride = sida_out_proj_bytes(d);
  p.bias_off = static_cast<size_t>(d) * d * 2;
  p.resid = resid; p.out = out;
  p.bf16_map = map; p.bf16_k = k;
  p.peer_bf16 = peers; p.peer_stride = peer_stride;
  p.err_flag = err_flag;
  const int cg = n_rows >= 1024 ? 2 : 1;
  // N tile 192 when it divides d: at d = 768 the 32K-row projection is 512
  // tiles (6.9 persistent rounds of 74 pairs) instead of 384 (5.2 rounds), and
  // this epilogue-bound GEMM gains more from the fuller last round than it
  // loses to the narrower tile (tools/proj_probe.py: 98 -> 92 us).
  // SIDA_OUTPROJ_BN=256|128 overrides (A/B).
  static int bn = -1;
  if (bn < 0) {
    const char* e = getenv("SIDA_OUTPROJ_BN");
    bn = e ? atoi(e) : 192;
  }
  if (bn == 192 && d % 192 == 0) {
    if (cg == 2) return sm100::launch_gemm<192, 2, 2>(ctx, wo_t, 1, p, 1, as_stream(stream));
    return sm100::launch_gemm<192, 2, 1>(ctx, wo_t, 1, p, 1, as_stream(stream));
  }
  if (bn == 128 && d % 128 == 0) {
    if (cg == 2) return sm100::launch_gemm<128, 2, 2>(ctx, wo_t, 1, p, 1, as_stream(stream));
    return sm100::launch_gemm<128, 2, 1>(ctx, wo_t, 1, p, 1, as_stream(stream));
  }
  return sm100::dispatch_gemm<2>(ctx, wo_t, 1, p, 1, cg, as_stream(stream));
}

// Return: the owner's grouped FFN writes each expert-output row (bf16, no
// alpha / residual -- the source combines) straight back into the SOURCE
// rank's buffer at its expert-sorted position: row_map[j] = src * peer_stride
// + row, peers[g] = rank g's return buffer.
extern "C" int sida_grouped_ffn_bf16_peer(const uint16_t* x_loc, int n_rows, int d, int h,
                                          const int32_t* off, int num_experts,
                                          const int32_t* expert_slot, const void* arena,
                                          size_t slot_stride, int n_slots, const int32_t* row_map,
                                          uint16_t* const* peers, int peer_stride,
                                          uint16_t* hidden, int32_t* err_flag, void* stream) {
  SIDA_REQUIRE(d % 64 == 0 && h % 64 == 0, SIDA_ERR_UNSUPPORTED,
               "tcgen05 FFN needs d, h multiples of 64 (d=%d h=%d)", d, h);
  SIDA_REQUIRE(n_rows >= 0 && num_experts >= 1 && num_experts <= sm100::kMaxListed &&
                   n_slots >= 1 && peer_stride >= 1,
               SIDA_ERR_CONTRACT, "bad ffn dims rows=%d K=%d slots=%d", n_rows, num_experts,
               n_slots);
  SIDA_REQUIRE(err_flag && hidden && x_loc && off && expert_slot && arena && row_map && peers,
               SIDA_ERR_CONTRACT, "null pointer passed to sida_grouped_ffn_bf16_peer");
  if (n_rows == 0) return SIDA_OK;
  cudaStream_t s = as_stream(stream);
  const uint8_t* ar = static_cast<const uint8_t*>(arena);
  const size_t w2_off = (size_t)h * d * 2, b1_off = 2 * w2_off, b2_off = b1_off + (size_t)h * 2;
  sm100::GemmParams p1{};
  p1.n_rows = n_rows; p1.kdim = d; p1.ndim = h;
  p1.off = off; p1.num_experts = num_experts; p1.expert_slot = expert_slot;
  p1.arena = ar; p1.slot_stride = slot_stride; p1.bias_off = b1_off;
  p1.hidden = hidden; p1.err_flag = err_flag;
  p1.half_tiles = 1;
  int st = sm100::dispatch_gemm<1>(x_loc, ar, n_slots, p1, num_experts,
                                   choose_cg(1, n_rows, num_experts), s);
  if (st) return st;
  sm100::GemmParams p2 = p1;
  p2.kdim = h; p2.ndim = d; p2.bias_off = b2_off;
  p2.row_map = row_map; p2.peer_bf16 = peers; p2.peer_stride = peer_stride;
  return sm100::dispatch_gemm<2>(hidden, ar + w2_off, n_slots, p2, num_experts,
                                 choose_cg(2, n_rows, num_experts), s);
}
