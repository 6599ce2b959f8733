// Expert FFN of one MoE layer as ONE persistent launch (sm_100a): both expert
// GEMMs, with the hidden activations passed from GEMM1 to GEMM2 through L2.
// Replaces ref moe.py:235-262 (moe_apply) for the many-expert shapes of the
// north star (Switch-base-64/128/256: a few hundred rows per expert).
//
// Tiles are swap-AB ("token-N"): the expert's weight rows are the UMMA M side
// (256 output features per CTA pair, tcgen05.mma.cta_group::2) and the
// expert's token rows the N side, one tile per expert up to kMaxTile rows
// (N = the row count rounded to 16, so an expert of 272 rows costs 272
// columns of MMA, not the 384 of two 256-row token tiles or the 512 of four
// 128-row ones), larger experts in balanced tiles of <= 256 rows.
//
// Work items, all the same MMA work (R x 256 x 3072 at d=768, h=3072):
//   G1(m, i): hidden[:, 1024 i .. +1024] = relu(X W1^T + b1) for token tile m,
//             four 256-feature sub-tiles back to back (K = d each)
//   G2(m, j): out[:, 256 j .. +256] = alpha (H W2^T + b2) + resid, unpermuted
//             through row_map (K = h)
// in the order G1 of m-tiles 0..lag-1, then per step s: G1(s), G2(s - lag),
// then the remaining G2s, dealt round-robin to the 74 CTA pairs. A G2 item's
// producer waits (acquire) until the 2 x n1 G1 epilogues of its m-tile have
// released their hidden rows; lag m-tiles of hidden (lag x 1.5 MB at 256
// rows) are in flight, so GEMM2 reads them from L2 and the 2 x N x h x 2 B
// hidden round trip through HBM disappears. The weights are loaded with an
// L2 evict-first policy so the stream of 9.4 MB expert images does not push
// the hidden rows out.
//
// TMEM (512 columns per CTA) is a ring of 16 chunks of 32 columns: a tile
// takes ceil(N/32) consecutive chunks (wrapping), so two 272-column tiles
// overlap their MMA and epilogue as soon as the first chunks of the older
// one are drained (the epilogue frees chunk by chunk). Each MMA covers at
// most 256 columns and never crosses the wrap; in cta_group::2 an MMA of N
// columns takes N/2 token rows from each CTA's shared memory, so CTA r holds
// the tile's token rows [r N/2, (r+1) N/2) contiguously and MMA piece k (n_k
// columns, B rows o_k .. o_k + n_k/2 in both CTAs) maps its column u to
// token o_k + u (u < n_k/2) or N/2 + o_k + u - n_k/2.
//
// CTA = 10 warps: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer
// (leader CTA), warps 2-9 epilogue (TMEM lane quarter x column-chunk parity).
// The G1->G2 flags carry an epoch tag read from a device counter that the
// last CTA of each launch advances, so they need no reset between launches
// and stay valid under CUDA-graph replay.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace sida {
namespace xffn {
using namespace sm100;

constexpr int BK = 64;                  // one SWIZZLE_128B row of bf16
constexpr int UMMA_K = 16;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kMaxTile = 320;           // tokens per tile (UMMA N over the pair)
constexpr int kSplitTile = 256;         // tile size bound above kMaxTile rows
constexpr int kBRows = kMaxTile / 2;    // token rows per CTA per stage
static_assert(kBRows % 32 == 0, "TMA boxes must tile the B stage");
constexpr int kBox = 32;                // token rows per TMA box (kBRows % kBox == 0)
constexpr uint32_t kABytes = 128 * BK * 2;
constexpr uint32_t kBBytes = kBRows * BK * 2;
constexpr uint32_t kBoxBytes = kBox * BK * 2;
constexpr int kStages = 6;
constexpr int kChunks = 16;             // TMEM ring: 16 x 32 columns
constexpr int kTileRing = 16;           // tile_full barriers (>= tiles in the ring)
constexpr int kSubs = 4;                // GEMM1 256-feature sub-tiles per item
constexpr int kMaxListed = 512;
constexpr int kMaxMTiles = 1 << 16;     // flag words per launch state

constexpr size_t smem_bytes() {
  return 1024 + kStages * (kABytes + kBBytes) + (2 * kStages + kTileRing + kChunks) * 8 + 16 +
         (2 * kMaxListed + 2) * 4;
}

struct Params {
  int n_rows, d, h;
  const int32_t* off;          // K+1 expert row offsets (permuted order)
  int num_experts;
  const int32_t* expert_slot;  // expert -> slot (-1: not resident -> err_flag)
  const int32_t* expert_list;  // optional subset
  int n_list;
  const uint8_t* arena;
  size_t slot_stride, b1_off, b2_off;
  uint16_t* hidden;            // (n_rows, h) bf16, L2-resident between the two halves
  const int32_t* row_map;      // output row of permuted row p
  const float* alpha;
  const float* resid;
  float* out;
  uint16_t* out_bf16;
  int32_t* err_flag;
  uint32_t* state;             // [0] epoch, [1] done CTAs, [2..] m-tile flags
  int lag;
  unsigned long long* prof;    // optional per-CTA cycle counters (SIDA_XFFN_PROF=1)
  int diag;                    // diagnostics: 1 = epilogue without math/stores
};

// prof slots per CTA: producer wait(empty), producer wait(flags), MMA wait(full),
// MMA wait(chunks), MMA total, epilogue wait(tile_full), epilogue total, prologue
constexpr int kProf = 8;
__device__ __forceinline__ unsigned long long clk() { return clock64(); }

// Token tiles of an expert with R rows: one tile up to kMaxTile rows, else
// balanced tiles of <= kSplitTile rows (multiples of 16).
__device__ __forceinline__ void tile_split(int R, int& base, int& count) {
  if (R <= 0) { base = 16; count = 0; return; }
  if (R <= kMaxTile) { base = R; count = 1; return; }
  const int n = ceil_div(R, kSplitTile);
  base = min(kSplitTile, (ceil_div(R, n) + 15) & ~15);
  count = ceil_div(R, base);
}

__device__ __forceinline__ int expert_row(const Params& p, int e) { return p.off[e]; }

struct Tile {
  bool g2;
  int mt, expert, row0, nrows, n16, f0, slot, ntiles;
};

// item order (see header): step s issues the n1 G1 items of m-tile s, then
// the n2 G2 items of m-tile s - lag
__device__ __forceinline__ void item_order(int t, int MT, int n1, int n2, int lag, bool& g2,
                                           int& mt, int& nt) {
  const int a = min(lag, MT);
  if (t < a * n1) { g2 = false; mt = t / n1; nt = t - mt * n1; return; }
  t -= a * n1;
  const int nb = (MT - a) * (n1 + n2);
  if (t < nb) {
    const int s = t / (n1 + n2), r = t - s * (n1 + n2);
    if (r < n1) { g2 = false; mt = a + s; nt = r; }
    else { g2 = true; mt = a + s - lag; nt = r - n1; }
    return;
  }
  t -= nb;
  g2 = true; mt = MT - a + t / n2; nt = t - (t / n2) * n2;
}

// L2 evict-first policy for the streamed expert weights
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void tma_w(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                      uint32_t mbar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(mbar), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint32_t idesc_m256(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(256 >> 4) << 24);
}

__global__ void __launch_bounds__(kThreads, 1)
expert_ffn_kernel(const __grid_constant__ CUtensorMap tmW1,  // (d, h, slot) box 64 x 128
                  const __grid_constant__ CUtensorMap tmW2,  // (h, d, slot) box 64 x 128
                  const __grid_constant__ CUtensorMap tmX,   // (d, n_rows) box 64 x 64
                  const __grid_constant__ CUtensorMap tmH,   // (h, n_rows) box 64 x 64
                  const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* tile_full = empty + kStages;
  uint64_t* chunk_empty = tile_full + kTileRing;
  uint32_t* s_misc = reinterpret_cast<uint32_t*>(chunk_empty + kChunks);  // tmem base, epoch
  int32_t* s_prefix = reinterpret_cast<int32_t*>(s_misc + 4);
  int32_t* s_expert = s_prefix + kMaxListed + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_list = p.expert_list ? p.n_list : p.num_experts;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int unit = blockIdx.x >> 1, n_units = gridDim.x >> 1;

  const unsigned long long t_entry = clk();
  if (warp == 2) {
    // token-tile prefix over the listed experts: one warp, 32 experts per step
    int acc = 0;
    for (int i0 = 0; i0 < n_list; i0 += 32) {
      const int i = i0 + lane;
      int cnt = 0, e = 0;
      if (i < n_list) {
        e = p.expert_list ? p.expert_list[i] : i;
        int base;
        tile_split(expert_row(p, e + 1) - expert_row(p, e), base, cnt);
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
    for (int i = 0; i < kTileRing; ++i) mbar_init(&tile_full[i], 1);
    for (int i = 0; i < kChunks; ++i) mbar_init(&chunk_empty[i], 2 * (kEpiWarps / 2));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmH)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_misc)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = s_misc[0];
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel's tail; its outputs (x_perm, residual) are read only after this
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) s_misc[1] = *reinterpret_cast<volatile uint32_t*>(p.state);
  __syncthreads();
  if (p.prof && threadIdx.x == 0) p.prof[blockIdx.x * kProf + 7] = clk() - t_entry;
  const uint32_t tag = (s_misc[1] + 1u) & 0xFFFFFFu;  // this launch's flag epoch

  const int MT = s_prefix[n_list];
  const int n_ft1 = p.h / 256;
  const int n1 = ceil_div(n_ft1, kSubs), n2 = p.d / 256;
  const int lag = max(1, p.lag);
  const int total = MT * (n1 + n2);
  const uint32_t flag_target = (tag << 8) | static_cast<uint32_t>(2 * n1);
  uint32_t* flags = p.state + 2;

  auto item = [&](int it, int& nsub, bool& g2, int& mt, int& nt) {
    item_order(it, MT, n1, n2, lag, g2, mt, nt);
    nsub = g2 ? 1 : min(kSubs, n_ft1 - nt * kSubs);
  };
  auto tile = [&](bool g2, int mt, int nt, int j) -> Tile {
    int lo = 0, hi = n_list - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_prefix[mid] <= mt) lo = mid; else hi = mid - 1;
    }
    Tile t;
    t.g2 = g2;
    t.mt = mt;
    t.expert = s_expert[lo];
    const int seg0 = expert_row(p, t.expert);
    const int R = expert_row(p, t.expert + 1) - seg0;
    int base, cnt;
    tile_split(R, base, cnt);
    const int q = mt - s_prefix[lo];
    t.row0 = seg0 + q * base;
    t.nrows = min(base, R - q * base);
    t.n16 = (t.nrows + 15) & ~15;
    t.f0 = g2 ? nt * 256 : (nt * kSubs + j) * 256;
    t.slot = p.expert_slot[t.expert];
    t.ntiles = cnt;
    return t;
  };

  if (warp == 0) {
    // ===== TMA producer (both CTAs): 128 weight rows + this CTA's half of the
    // tokens; the warp walks the schedule in lockstep, one elected lane issues
    {
      // experts held by one token tile stream their weights once: evict-first;
      // experts split over several tiles re-read them: normal policy
      const uint64_t pol_first = evict_first_policy();
      uint64_t pol_normal;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_normal));
      int stage = 0;
      uint32_t phase = 0;
      unsigned long long w_empty = 0, w_flag = 0;
      for (int it = unit; it < total; it += n_units) {
        int nsub, mt, nt;
        bool g2;
        item(it, nsub, g2, mt, nt);
        for (int j = 0; j < nsub; ++j) {
          const Tile t = tile(g2, mt, nt, j);
          if (t.slot < 0) continue;
          if (g2 && j == 0) {
            // the hidden rows of this m-tile: every G1 epilogue of both CTAs released
            uint32_t v;
            const unsigned long long c0 = p.prof ? clk() : 0;
            while (true) {
              asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flags + mt) : "memory");
              if (__shfl_sync(0xffffffffu, v, 0) == flag_target) break;
              __nanosleep(32);
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
            if (p.prof) w_flag += clk() - c0;
          }
          const int half = t.n16 >> 1;
          const int nbox = ceil_div(half, kBox);
          const int xrow = t.row0 + static_cast<int>(rank) * half;
          const CUtensorMap* tw = g2 ? &tmW2 : &tmW1;
          const CUtensorMap* tx = g2 ? &tmH : &tmX;
          const int nkb = (g2 ? p.h : p.d) / BK;
          const uint64_t pol = t.ntiles == 1 ? pol_first : pol_normal;
          for (int kb = 0; kb < nkb; ++kb) {
            const unsigned long long c1 = p.prof ? clk() : 0;
            mbar_wait(&empty[stage], phase ^ 1);
            if (p.prof) w_empty += clk() - c1;
            const uint32_t fb = map_rank(smem_u32(&full[stage]), 0);
            if (elect_one()) {
              if (leader) mbar_expect_tx(&full[stage], 2 * (kABytes + nbox * kBoxBytes));
              tma_w(sA + stage * kABytes, tw, kb * BK, t.f0 + static_cast<int>(rank) * 128,
                    t.slot, fb, pol);
              for (int b = 0; b < nbox; ++b)
                tma_load_2d<2>(sB + stage * kBBytes + b * kBoxBytes, tx, kb * BK,
                               xrow + b * kBox, fb);
            }
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
      if (p.prof && lane == 0) {
        p.prof[blockIdx.x * kProf + 0] = w_empty;
        p.prof[blockIdx.x * kProf + 1] = w_flag;
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA): warp-uniform walk, one elected lane issues
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t chunk_par = 0;  // bit c: parity of chunk c's next release
      int pos = 0;             // ring position (chunk index) of the next tile
      int tcount = 0;
      unsigned long long w_full = 0, w_chunk = 0;
      const unsigned long long m0 = p.prof ? clk() : 0;
      for (int it = unit; it < total; it += n_units) {
        int nsub, mt, nt;
        bool g2;
        item(it, nsub, g2, mt, nt);
        for (int j = 0; j < nsub; ++j) {
          const Tile t = tile(g2, mt, nt, j);
          if (t.slot < 0) {
            if (lane == 0) atomicExch(p.err_flag, 1);
            continue;
          }
          const int nch = (t.n16 + 31) >> 5;
          const unsigned long long c2 = p.prof ? clk() : 0;
          for (int i = 0; i < nch; ++i) {
            const int c = (pos + i) & (kChunks - 1);
            mbar_wait_cluster(&chunk_empty[c], ((chunk_par >> c) & 1u) ^ 1u);
            chunk_par ^= 1u << c;
          }
          if (p.prof) w_chunk += clk() - c2;
          tc_fence_after();
          const int nkb = (g2 ? p.h : p.d) / BK;
          for (int kb = 0; kb < nkb; ++kb) {
            const unsigned long long c3 = p.prof ? clk() : 0;
            mbar_wait(&full[stage], phase);
            if (p.prof) w_full += clk() - c3;
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + stage * kABytes);
            const uint32_t b0 = smem_u32(sB + stage * kBBytes);
            if (elect_one()) {
              int col = pos * 32, rem = t.n16, o = 0;
              while (rem > 0) {
                const int n = min(rem, min(256, 512 - col));
                const uint32_t idesc = idesc_m256(n);
#pragma unroll
                for (int k = 0; k < BK / UMMA_K; ++k)
                  umma_bf16<2>(tmem_base + col, sw128_desc(a0 + k * UMMA_K * 2),
                               sw128_desc(b0 + o * 128 + k * UMMA_K * 2), idesc, (kb | k) != 0);
                o += n >> 1;
                rem -= n;
                col = (col + n) & 511;
              }
              tc_commit<2>(&empty[stage]);
            }
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
          if (elect_one()) tc_commit<2>(&tile_full[tcount & (kTileRing - 1)]);
          __syncwarp();
          ++tcount;
          pos = (pos + nch) & (kChunks - 1);
        }
      }
      if (p.prof && lane == 0) {
        unsigned long long* pr = p.prof + blockIdx.x * kProf;
        pr[2] = w_full;
        pr[3] = w_chunk;
        pr[4] = clk() - m0;
      }
    }
  } else {
    // ===== epilogue: warp owns TMEM lanes 32 (w % 4) .. (32 of this CTA's 128
    // features) and the tile's 32-column chunks of one parity
    const int quarter = warp & 3;
    const int parity = (warp - 2) >> 2;
    int pos = 0, tcount = 0;
    unsigned long long w_tf = 0;
    const unsigned long long e0 = p.prof ? clk() : 0;
    for (int it = unit; it < total; it += n_units) {
      int nsub, mt, nt;
      bool g2;
      item(it, nsub, g2, mt, nt);
      bool any = false;
      for (int j = 0; j < nsub; ++j) {
        const Tile t = tile(g2, mt, nt, j);
        if (t.slot < 0) continue;
        any = true;
        const int nch = (t.n16 + 31) >> 5;
        const int f = t.f0 + static_cast<int>(rank) * 128 + quarter * 32 + lane;
        const uint16_t* bias = reinterpret_cast<const uint16_t*>(
            p.arena + static_cast<size_t>(t.slot) * p.slot_stride + (g2 ? p.b2_off : p.b1_off));
        const float b = bf16_to_f32(bias[f]);
        const int ndim = g2 ? p.d : p.h;
        const int halfN = t.n16 >> 1;
        const unsigned long long c4 = p.prof ? clk() : 0;
        mbar_wait(&tile_full[tcount & (kTileRing - 1)], (tcount / kTileRing) & 1);
        if (p.prof) w_tf += clk() - c4;
        tc_fence_after();
        for (int c = parity; c < nch; c += 2) {
          // the MMA piece holding tile columns [32 c, 32 c + 32): pieces start at
          // chunk boundaries and never cross the ring wrap or 256 columns
          int col = pos * 32, rem = t.n16, o = 0, s0 = 0, pn = 0, po = 0;
          while (rem > 0) {
            const int n = min(rem, min(256, 512 - col));
            if (32 * c >= s0 && 32 * c < s0 + n) { pn = n; po = o; break; }
            s0 += n; o += n >> 1; rem -= n; col = (col + n) & 511;
          }
          const int ch = (pos + c) & (kChunks - 1);
          uint32_t v[32];
          tmem_ld32_nowait(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + ch * 32, v);
          // token of column 32 c + j: u = 32 c + j - s0 within the piece
          const int u0 = 32 * c - s0, hp = pn >> 1;
          auto tok_of = [&](int jj) -> int {
            const int u = u0 + jj;
            if (u >= pn) return 1 << 30;  // beyond the tile's last piece
            return u < hp ? po + u : halfN + po + (u - hp);
          };
          // the chunk's values are in registers once the load completes: hand
          // this warp's quarter of it back to the MMA issuer before the math
          auto release = [&]() {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(map_rank(smem_u32(&chunk_empty[ch]), 0));
          };
          if (p.diag == 1 || (p.diag == 2 && g2) || (p.diag == 3 && !g2)) {
            tmem_wait_ld();
            release();
          } else if (!g2) {
            tmem_wait_ld();
            release();
            const bool odd = lane & 1;
#pragma unroll
            for (int jj = 0; jj < 32; jj += 2) {
              const float y0 = fmaxf(__uint_as_float(v[jj]) + b, 0.f);
              const float y1 = fmaxf(__uint_as_float(v[jj + 1]) + b, 0.f);
              const float other = __shfl_xor_sync(0xffffffffu, odd ? y0 : y1, 1);
              const uint32_t w = odd ? bf16x2_rn(other, y1) : bf16x2_rn(y0, other);
              const int tk = tok_of(jj + (odd ? 1 : 0));
              if (tk < t.nrows)
                *reinterpret_cast<uint32_t*>(p.hidden + static_cast<size_t>(t.row0 + tk) * ndim +
                                             (f & ~1)) = w;
            }
          } else {
            // lane jj holds token tok_of(jj)'s output row and alpha; broadcast by shuffles
            const int my_tok = tok_of(lane);
            const bool my_valid = my_tok < t.nrows;
            int orow_l = 0;
            float a_l = 1.f;
            if (my_valid) {
              orow_l = p.row_map ? p.row_map[t.row0 + my_tok] : t.row0 + my_tok;
              if (p.alpha) a_l = p.alpha[t.row0 + my_tok];
            }
            const unsigned vmask = __ballot_sync(0xffffffffu, my_valid);
            float x[32];
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              const int orow = __shfl_sync(0xffffffffu, orow_l, jj);
              x[jj] = (p.resid && ((vmask >> jj) & 1u))
                          ? __ldg(p.resid + static_cast<size_t>(orow) * ndim + f)
                          : 0.f;
            }
            tmem_wait_ld();
            release();
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              const int orow = __shfl_sync(0xffffffffu, orow_l, jj);
              const float a = __shfl_sync(0xffffffffu, a_l, jj);
              if ((vmask >> jj) & 1u) {
                const float y = x[jj] + (__uint_as_float(v[jj]) + b) * a;
                const size_t at = static_cast<size_t>(orow) * ndim + f;
                if (p.out) p.out[at] = y;
                if (p.out_bf16) p.out_bf16[at] = __bfloat16_as_ushort(__float2bfloat16_rn(y));
              }
            }
          }
        }
        ++tcount;
        pos = (pos + nch) & (kChunks - 1);
      }
      if (!g2 && any) {
        // this CTA's hidden columns of G1 item (mt, nt) are stored: make them
        // visible at gpu scope, then count the release for the G2 producers
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        if (warp == 2 && lane == 0) {
          uint32_t old = atomicAdd(flags + mt, 0u), want;
          do {
            want = ((old >> 8) == tag) ? old + 1u : ((tag << 8) | 1u);
            const uint32_t seen = atomicCAS(flags + mt, old, want);
            if (seen == old) break;
            old = seen;
          } while (true);
        }
      }
    }
    if (p.prof && warp == 2 && lane == 0) {
      p.prof[blockIdx.x * kProf + 5] = w_tf;
      p.prof[blockIdx.x * kProf + 6] = clk() - e0;
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512));
  }
  if (threadIdx.x == 0) {
    // the last CTA of the launch advances the epoch for the next one
    __threadfence();
    if (atomicAdd(p.state + 1, 1u) == gridDim.x - 1) {
      p.state[1] = 0;
      __threadfence();
      atomicAdd(p.state, 1u);
    }
  }
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

static int map_nd(CUtensorMap* m, int rank, const void* base, const cuuint64_t* dims,
                  const cuuint64_t* strides, const cuuint32_t* box) {
  auto fn = encode_fn();
  SIDA_REQUIRE(fn, SIDA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SIDA_REQUIRE(r == CUDA_SUCCESS, SIDA_ERR_CUDA, "tensor map encode failed: %d", (int)r);
  return SIDA_OK;
}

// Launch state (epoch, done counter, m-tile flags) per (device, stream),
// zeroed once when first used (outside any graph capture: the engine warms up
// every shape before capturing it).
static int launch_state(cudaStream_t s, uint32_t** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, uint32_t*> states;
  int dev = 0;
  SIDA_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto& slot = states[{dev, s}];
  if (!slot) {
    const size_t bytes = (2 + static_cast<size_t>(kMaxMTiles)) * sizeof(uint32_t);
    SIDA_CUDA(cudaMalloc(&slot, bytes));
    SIDA_CUDA(cudaMemset(slot, 0, bytes));
    SIDA_CUDA(cudaDeviceSynchronize());
  }
  *out = slot;
  return SIDA_OK;
}

static int g_lag = -1;
static unsigned long long* g_prof = nullptr;

}  // namespace xffn
}  // namespace sida

using namespace sida;

// Observability: the per-CTA cycle counters of the last one-launch FFN
// (SIDA_XFFN_PROF=1) into out[148][8]; synchronises the device.
extern "C" int sida_debug_xffn_prof(unsigned long long* out) {
  using namespace sida::xffn;
  SIDA_REQUIRE(g_prof, SIDA_ERR_UNSUPPORTED, "run with SIDA_XFFN_PROF=1");
  SIDA_CUDA(cudaDeviceSynchronize());
  SIDA_CUDA(cudaMemcpy(out, g_prof, kNumSMs * kProf * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost));
  return SIDA_OK;
}

// Applicability of the one-launch expert FFN (sida_grouped_ffn_bf16 routes
// here when this returns 1): d a multiple of 256 and h of 1024.
extern "C" int sida_expert_ffn_applicable(int d, int h) {
  return d % 256 == 0 && h % 1024 == 0 && d >= 256 && h >= 1024;
}

extern "C" int sida_expert_ffn_launch(const uint16_t* x_perm, int n_rows, int d, int h,
                                      const int32_t* off, int num_experts,
                                      const int32_t* expert_slot, const int32_t* expert_list,
                                      int n_list, const void* arena, size_t slot_stride,
                                      int n_slots, const int32_t* row_map, const float* alpha,
                                      const float* resid, float* out, uint16_t* out_bf16,
                                      uint16_t* hidden, int32_t* err_flag, void* stream) {
  using namespace sida::xffn;
  SIDA_REQUIRE(sida_expert_ffn_applicable(d, h), SIDA_ERR_UNSUPPORTED,
               "expert FFN launch needs d %% 256 == 0 and h %% 1024 == 0 (d=%d h=%d)", d, h);
  const int listed = expert_list ? n_list : num_experts;
  SIDA_REQUIRE(listed <= kMaxListed, SIDA_ERR_UNSUPPORTED, "more than %d experts listed",
               kMaxListed);
  SIDA_REQUIRE(ceil_div(n_rows, 16) + listed <= kMaxMTiles, SIDA_ERR_UNSUPPORTED,
               "too many token tiles (%d rows)", n_rows);
  if (n_rows == 0 || listed == 0) return SIDA_OK;
  cudaStream_t s = as_stream(stream);
  static bool configured = false;
  if (!configured) {
    SIDA_CUDA(cudaFuncSetAttribute(expert_ffn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_bytes()));
    configured = true;
  }
  if (g_lag < 0) {
    const char* e = getenv("SIDA_XFFN_LAG");
    g_lag = e ? atoi(e) : 25;
  }
  const uint8_t* ar = static_cast<const uint8_t*>(arena);
  const size_t w2_off = (size_t)h * d * 2, b1_off = 2 * w2_off, b2_off = b1_off + (size_t)h * 2;
  CUtensorMap tw1, tw2, tx, th;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)h, (cuuint64_t)n_slots};
    const cuuint64_t str[2] = {(cuuint64_t)d * 2, (cuuint64_t)slot_stride};
    const cuuint32_t box[3] = {BK, 128, 1};
    int st = map_nd(&tw1, 3, ar, dims, str, box);
    if (st) return st;
  }
  {
    const cuuint64_t dims[3] = {(cuuint64_t)h, (cuuint64_t)d, (cuuint64_t)n_slots};
    const cuuint64_t str[2] = {(cuuint64_t)h * 2, (cuuint64_t)slot_stride};
    const cuuint32_t box[3] = {BK, 128, 1};
    int st = map_nd(&tw2, 3, ar + w2_off, dims, str, box);
    if (st) return st;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n_rows};
    const cuuint64_t str[1] = {(cuuint64_t)d * 2};
    const cuuint32_t box[2] = {BK, kBox};
    int st = map_nd(&tx, 2, x_perm, dims, str, box);
    if (st) return st;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)h, (cuuint64_t)n_rows};
    const cuuint64_t str[1] = {(cuuint64_t)h * 2};
    const cuuint32_t box[2] = {BK, kBox};
    int st = map_nd(&th, 2, hidden, dims, str, box);
    if (st) return st;
  }
  uint32_t* state = nullptr;
  int st = launch_state(s, &state);
  if (st) return st;
  Params p{};
  p.n_rows = n_rows; p.d = d; p.h = h;
  p.off = off; p.num_experts = num_experts; p.expert_slot = expert_slot;
  p.expert_list = expert_list; p.n_list = n_list;
  p.arena = ar; p.slot_stride = slot_stride; p.b1_off = b1_off; p.b2_off = b2_off;
  p.hidden = hidden; p.row_map = row_map; p.alpha = alpha; p.resid = resid;
  p.out = out; p.out_bf16 = out_bf16; p.err_flag = err_flag; p.state = state; p.lag = g_lag;
  if (const char* e = getenv("SIDA_XFFN_DIAG")) p.diag = atoi(e);
  static int prof_on = -1;
  if (prof_on < 0) {
    const char* e = getenv("SIDA_XFFN_PROF");
    prof_on = e ? atoi(e) : 0;
  }
  if (prof_on) {
    if (!g_prof) SIDA_CUDA(cudaMalloc(&g_prof, kNumSMs * kProf * sizeof(unsigned long long)));
    SIDA_CUDA(cudaMemsetAsync(g_prof, 0, kNumSMs * kProf * sizeof(unsigned long long), s));
    p.prof = g_prof;
  }

  const int max_items = (ceil_div(n_rows, 16) + listed) * (h / 1024 + d / 256);
  const int units = std::max(1, std::min(max_items, kNumSMs / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(units * 2);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes();
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  const char* pe = getenv("SIDA_PDL");
  attr[1].val.programmaticStreamSerializationAllowed = pe ? atoi(pe) : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  SIDA_CUDA(cudaLaunchKernelEx(&cfg, expert_ffn_kernel, tw1, tw2, tx, th, p));
  count_launch();
  return SIDA_OK;
}
