// Fused mixing-attention core on the 5th-gen tensor cores (sm_100a):
//   ctx = softmax(q k^T / sqrt(d)) v        per sequence, single head, non-causal
// for sequences of at most 512 tokens (ref moe.py:220-233; the projections
// q,k,v = x W and the output projection run as GEMMs around this kernel).
//
// Up to 128 tokens: one CTA per sequence, two CTAs per SM (~105 KB smem, 256
// TMEM columns each), so a 256-sequence batch is resident in a single wave.
// Up to 256 tokens: one CTA per (sequence, 128-query block) over all the
// sequence's keys (S is 128 x 256 in TMEM, P 64 KB), one CTA per SM. Inside
// a CTA (shown for 128 keys):
//
//   phase 1  S = Q K^T (M=128 queries, N=128 keys, K=d) with tcgen05.mma,
//            Q and K k-blocks streamed by TMA through a 2-slot ring,
//            accumulator in TMEM columns [0, 128)
//   phase 2  softmax rows (4 warps, thread = query row): row max of the
//            scaled scores over the sequence's keys, e = exp(s/sqrt(d) - m)
//            written as bf16 straight into the K-major SWIZZLE_128B layout
//            of the next MMA's A operand; 1/sum kept in a register
//   phase 3  C = P V in d-chunks of 128 columns (V read MN-major: the token
//            rows of qkv are the K dimension), TMEM double buffer
//            {[128,256), [0,128)} so the epilogue of chunk j overlaps the
//            MMAs of chunk j+1; epilogue scales by 1/sum, rounds to bf16 and
//            stores through a swizzled smem transpose (coalesced 64 B rows).
//
// Keys past the sequence end are masked (their TMA rows belong to the next
// sequence or are zero-filled past the batch), query rows past it are
// computed and dropped. softmax(s) V = (e V) / sum: normalising after the
// product instead of before is exact in real arithmetic; both forms round P
// to bf16 once.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace sida {
namespace attn {

using namespace sm100;

constexpr int BM = 128;        // queries per CTA (one TMEM lane each)
constexpr int BK = 64;         // d per phase-1 k-block (one SW128 row)
constexpr int NC = 128;        // d columns per phase-3 chunk (64 when d % 128 != 0)
constexpr int kSlots = 2;
constexpr int kStageTile = 32 * 32 * 2; // per-warp bf16 epilogue staging tile
constexpr int kEpiWarps = 4;
constexpr int kThreads = 64 + 32 * kEpiWarps;

// Per key-count variant (NKEY = keys per CTA = the longest sequence served):
//   128: ring slot 32 KB (Q 16 + K 16 KB, or a V chunk 2 x 16 KB), P 32 KB,
//        TMEM 256 columns (S [0,128), C chunks {[128,256), [0,128)}), 2 CTAs/SM
//   256: ring slot 64 KB (Q 16 + K 32 KB, or a V chunk 2 x 32 KB), P 64 KB,
//        TMEM 512 columns (S [0,256), C chunks {[256,384), [384,512)}), 1 CTA/SM
//   512: ring slot 80 KB (Q 16 + K 64 KB, or half a V chunk: 256 keys x 2 x 64
//        columns), S fills all 512 TMEM columns (two N=256 MMAs per k-step) and
//        P stays in TMEM: the softmax warps write bf16 P pairs over S's first
//        256 columns (tcgen05.st, each lane only overwriting scores it has
//        already read) and C = P V reads A from TMEM (the tcgen05 "TS" form),
//        so the 128 KB P tile never touches shared memory; C chunks use the
//        consumed S columns {[256,384), [384,512)}. 1 CTA/SM.
template <int NKEY, int NCT = NC>
struct Cfg {
  static constexpr bool kPT = NKEY == 512;                // P in TMEM
  static constexpr int kVKeys = kPT ? 256 : NKEY;         // keys per V stage
  static constexpr int kVPerChunk = NKEY / kVKeys;        // V stages per d chunk
  static constexpr int kQKBytes = BM * 128 + NKEY * 128;
  static constexpr int kVBytes = kVKeys * NCT * 2;
  static constexpr int kSlot = kQKBytes > kVBytes ? kQKBytes : kVBytes;
  static constexpr int kPBytes = kPT ? 0 : BM * NKEY * 2;  // NKEY/64 K-atoms x 128 rows x 128 B
  static constexpr int kSN = NKEY > 256 ? 256 : NKEY;     // N of one phase-1 MMA
  static constexpr uint32_t kTmemCols = NKEY == 128 ? 256 : 512;
  static constexpr uint32_t kC0 = NKEY == 128 ? 128 : 256;  // C chunk buffers (TMEM columns)
  static constexpr uint32_t kC1 = NKEY == 128 ? 0 : 384;
  static constexpr int kMinBlocks = NKEY == 128 ? 2 : 1;
  static constexpr size_t kSmem = 1024 + kSlots * kSlot + kPBytes + kEpiWarps * kStageTile + 256;
};

// SWIZZLE_128B MN-major operand: 64-element MN groups `lbo` bytes apart, 8-row
// K groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr, uint32_t lbo) {
  uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int NKEY, int NCT>
__global__ void __launch_bounds__(kThreads, Cfg<NKEY, NCT>::kMinBlocks)
attn_core_kernel(const __grid_constant__ CUtensorMap tm_qkv, const int32_t* __restrict__ seq_off,
                 int d, float scale_log2e, uint16_t* __restrict__ ctx) {
  using C = Cfg<NKEY, NCT>;
  constexpr int kSlot = C::kSlot;
  constexpr int kPBytes = C::kPBytes;
  constexpr uint32_t kTmemCols = C::kTmemCols;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint8_t* sP = ring + kSlots * kSlot;
  uint8_t* sOut = sP + kPBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + kEpiWarps * kStageTile);
  uint64_t* full = bars;              // [kSlots]
  uint64_t* empty = bars + kSlots;    // [kSlots]
  uint64_t* s_full = bars + 2 * kSlots;
  uint64_t* p_full = s_full + 1;
  uint64_t* c_full = p_full + 1;      // [2]
  uint64_t* c_empty = c_full + 2;     // [2]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(c_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seq = blockIdx.x;
  const int row0 = seq_off[seq];              // first key / token of the sequence
  const int T = seq_off[seq + 1] - row0;
  const int q0 = blockIdx.y * BM;             // first query row of this CTA (in the sequence)
  if (q0 >= T) return;                        // (uniform: before any barrier / TMEM use)
  const int n_kb = d / BK, n_chunks = d / NCT;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, kEpiWarps);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&c_full[i], 1);
      mbar_init(&c_empty[i], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_qkv)) : "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  // let the output projection (launched with programmatic serialization)
  // start its prologue while this grid drains; this grid is itself launched
  // that way behind the QKV GEMM, so everything above overlapped that GEMM's
  // tail and qkv is read only after it has completed
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    // ===== TMA producer: 12 (Q, K) k-blocks, then d/NC V chunks, one ring
    // (the warp walks the ring in lockstep, one elected lane issues)
    {
      int slot = 0;
      uint32_t phase = 0;
      const int n_loads = n_kb + n_chunks * C::kVPerChunk;
      for (int i = 0; i < n_loads; ++i) {
        mbar_wait(&empty[slot], phase ^ 1);
        uint8_t* dst = ring + slot * kSlot;
        const uint32_t fb = smem_u32(&full[slot]);
        if (!elect_one()) {
        } else if (i < n_kb) {
          mbar_expect_tx(&full[slot], C::kQKBytes);
          tma_load_2d<1>(dst, &tm_qkv, i * BK, row0 + q0, fb);              // Q rows
#pragma unroll
          for (int kh = 0; kh < NKEY / 128; ++kh)                           // K rows
            tma_load_2d<1>(dst + BM * 128 + kh * 128 * 128, &tm_qkv, d + i * BK,
                           row0 + kh * 128, fb);
        } else {
          mbar_expect_tx(&full[slot], C::kVBytes);
          const int vi = i - n_kb;
          const int c0 = 2 * d + (vi / C::kVPerChunk) * NCT;
          const int k0 = row0 + (vi % C::kVPerChunk) * C::kVKeys;
#pragma unroll
          for (int gcol = 0; gcol < NCT / 64; ++gcol)                       // V[:, c0 + 64 g ..]
#pragma unroll
            for (int kh = 0; kh < C::kVKeys / 128; ++kh)
              tma_load_2d<1>(dst + gcol * (C::kVKeys * 128) + kh * 128 * 128, &tm_qkv,
                             c0 + gcol * 64, k0 + kh * 128, fb);
        }
        __syncwarp();
        if (++slot == kSlots) { slot = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: warp-uniform walk, one elected lane issues the MMAs
    // and their commits (descriptors in uniform registers)
    {
      constexpr uint32_t idesc_s = idesc_bf16<BM, C::kSN>();
      constexpr uint32_t idesc_c = idesc_bf16<BM, NCT>() | (1u << 16);  // B (V) MN-major
      int slot = 0;
      uint32_t phase = 0;
      for (int i = 0; i < n_kb; ++i) {
        mbar_wait(&full[slot], phase);
        tc_fence_after();
        const uint32_t a0 = smem_u32(ring + slot * kSlot);
        const uint32_t b0 = a0 + BM * 128;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
#pragma unroll
            for (int nh = 0; nh < NKEY / C::kSN; ++nh)  // 512 keys: two N=256 halves
              umma_bf16<1>(tmem + nh * C::kSN, sw128_desc(a0 + k * 32),
                           sw128_desc(b0 + nh * C::kSN * 128 + k * 32), idesc_s, (i | k) != 0);
          tc_commit<1>(&empty[slot]);
        }
        __syncwarp();
        if (++slot == kSlots) { slot = 0; phase ^= 1; }
      }
      if (elect_one()) tc_commit<1>(s_full);
      __syncwarp();
      mbar_wait(p_full, 0);  // P in smem (and S fully read: its TMEM columns free)
      tc_fence_after();
      const uint32_t p0 = smem_u32(sP);
      for (int j = 0; j < n_chunks; ++j) {
        const int b = j & 1;
        if (j >= 2) mbar_wait(&c_empty[b], ((j >> 1) - 1) & 1);
        const uint32_t d_tmem = tmem + (b == 0 ? C::kC0 : C::kC1);
        for (int hv = 0; hv < C::kVPerChunk; ++hv) {
          mbar_wait(&full[slot], phase);
          tc_fence_after();
          const uint32_t v0 = smem_u32(ring + slot * kSlot);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < C::kVKeys / 16; ++k) {  // 16 keys per MMA, V rows 16k..
              const uint64_t vb = sw128_mn_desc(v0 + k * 16 * 128, C::kVKeys * 128);
              if constexpr (C::kPT)  // P from TMEM: keys hv*256 + 16k.. = columns /2
                umma_bf16_ts(d_tmem, tmem + hv * (C::kVKeys / 2) + k * 8, vb, idesc_c,
                             (hv | k) != 0);
              else                   // P from smem: atom k/4, 16-key step k%4
                umma_bf16<1>(d_tmem, sw128_desc(p0 + (k >> 2) * (BM * 128) + (k & 3) * 32), vb,
                             idesc_c, k != 0);
            }
            tc_commit<1>(&empty[slot]);
          }
          __syncwarp();
          if (++slot == kSlots) { slot = 0; phase ^= 1; }
        }
        if (elect_one()) tc_commit<1>(&c_full[b]);
        __syncwarp();
      }
    }
  } else {
    // ===== softmax + epilogue: warp w owns TMEM lanes / query rows 32*(w%4)..
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // query row within the CTA
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    mbar_wait(s_full, 0);
    tc_fence_after();
    uint32_t v[32];
    float m = -INFINITY;
#pragma unroll
    for (int c = 0; c < NKEY / 32; ++c) {
      tmem_ld32_nowait(t_lane + c * 32, v);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c * 32 + j < T) m = fmaxf(m, __uint_as_float(v[j]));
    }
    const float mb = m * scale_log2e;
    float sum = 0.f;
    const uint32_t prow = smem_u32(sP) + r * 128;
#pragma unroll
    for (int c = 0; c < NKEY / 32; ++c) {
      tmem_ld32_nowait(t_lane + c * 32, v);
      tmem_wait_ld();
      float e[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        e[j] = c * 32 + j < T ? exp2f(fmaf(__uint_as_float(v[j]), scale_log2e, -mb)) : 0.f;
        sum += e[j];
      }
      if constexpr (C::kPT) {
        // keys c*32 .. +31 -> bf16 pairs in columns c*16 .. +15 of this lane
        // (scores of keys < c*32 + 32 are already read: no lane overwrites an
        // unread score)
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) pk[q] = bf16x2_rn(e[2 * q], e[2 * q + 1]);
        tmem_st16(t_lane + c * 16, pk);
      } else {
        // keys c*32 .. +31 = atom c/2, 16-B chunks 4*(c%2) .. +3 of row r
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 o;
          o.x = bf16x2_rn(e[q * 8 + 0], e[q * 8 + 1]);
          o.y = bf16x2_rn(e[q * 8 + 2], e[q * 8 + 3]);
          o.z = bf16x2_rn(e[q * 8 + 4], e[q * 8 + 5]);
          o.w = bf16x2_rn(e[q * 8 + 6], e[q * 8 + 7]);
          const int chunk = (c & 1) * 4 + q;
          sts128(prow + (c >> 1) * (BM * 128) + ((chunk ^ (r & 7)) << 4), o);
        }
      }
    }
    const float inv_sum = 1.f / sum;
    if constexpr (C::kPT) tmem_wait_st();                           // P -> tensor core (TMEM)
    else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P -> tensor core (smem)
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_local(p_full);

    // epilogue: chunk j of C -> bf16 ctx rows, through a swizzled 32x32 tile
    const uint32_t stile = smem_u32(sOut + (warp - 2) * kStageTile);
    const int q_row0 = row0 + q0 + quarter * 32;  // first global row of this warp
    for (int j = 0; j < n_chunks; ++j) {
      const int b = j & 1;
      mbar_wait(&c_full[b], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t t_c = t_lane + (b == 0 ? C::kC0 : C::kC1);
#pragma unroll
      for (int c = 0; c < NCT / 32; ++c) {
        tmem_ld32_nowait(t_c + c * 32, v);
        tmem_wait_ld();
        const uint32_t srow = stile + lane * 64;
        const int sw = (lane >> 1) & 3;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 o;
          o.x = bf16x2_rn(__uint_as_float(v[q * 8 + 0]) * inv_sum,
                          __uint_as_float(v[q * 8 + 1]) * inv_sum);
          o.y = bf16x2_rn(__uint_as_float(v[q * 8 + 2]) * inv_sum,
                          __uint_as_float(v[q * 8 + 3]) * inv_sum);
          o.z = bf16x2_rn(__uint_as_float(v[q * 8 + 4]) * inv_sum,
                          __uint_as_float(v[q * 8 + 5]) * inv_sum);
          o.w = bf16x2_rn(__uint_as_float(v[q * 8 + 6]) * inv_sum,
                          __uint_as_float(v[q * 8 + 7]) * inv_sum);
          sts128(srow + ((q ^ sw) << 4), o);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rr = i * 8 + (lane >> 2), q = lane & 3;
          const uint4 val = lds128(stile + rr * 64 + ((q ^ ((rr >> 1) & 3)) << 4));
          if (q0 + quarter * 32 + rr < T)
            *reinterpret_cast<uint4*>(ctx + static_cast<size_t>(q_row0 + rr) * d + j * NCT +
                                      c * 32 + q * 8) = val;
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&c_empty[b]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

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

template <int NKEY, int NCT>
static int launch_core(const CUtensorMap& tm, const int32_t* seq_off, int n_seq, int nq, int d,
                       float scale_log2e, uint16_t* ctx, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    SIDA_CUDA(cudaFuncSetAttribute(attn_core_kernel<NKEY, NCT>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)Cfg<NKEY, NCT>::kSmem));
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_seq, nq);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg<NKEY, NCT>::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SIDA_CUDA(cudaLaunchKernelEx(&cfg, attn_core_kernel<NKEY, NCT>, tm, seq_off, d, scale_log2e,
                               ctx));
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

}  // namespace attn
}  // namespace sida

using namespace sida;

// qkv: bf16 (n_tokens, 3d) = [q | k | v] per token (x @ [Wq|Wk|Wv]);
// seq_off: int32 (n_seq + 1) exclusive offsets on the concatenated token axis;
// every sequence at most 512 tokens; ctx: bf16 (n_tokens, d).
extern "C" int sida_attention_core(const uint16_t* qkv, const int32_t* seq_off, int n_seq,
                                   int n_tokens, int max_len, int d, uint16_t* ctx,
                                   void* stream) {
  SIDA_REQUIRE(d % 64 == 0 && d >= 64, SIDA_ERR_UNSUPPORTED,
               "fused attention needs d multiple of 64 (d=%d)", d);
  SIDA_REQUIRE(max_len >= 1 && max_len <= 512, SIDA_ERR_UNSUPPORTED,
               "fused attention handles sequences of at most 512 tokens (got %d)", max_len);
  SIDA_REQUIRE(n_seq >= 0 && n_tokens >= 0, SIDA_ERR_CONTRACT, "bad attention dims");
  SIDA_REQUIRE(qkv && seq_off && ctx, SIDA_ERR_CONTRACT,
               "null pointer passed to sida_attention_core");
  if (n_seq == 0 || n_tokens == 0) return SIDA_OK;
  auto fn = attn::encode_fn();
  SIDA_REQUIRE(fn, SIDA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap tm;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(3 * d), static_cast<cuuint64_t>(n_tokens)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(3 * d) * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(qkv), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SIDA_REQUIRE(r == CUDA_SUCCESS, SIDA_ERR_CUDA, "tensor map encode failed: %d", (int)r);
  const float scale_log2e = 1.4426950408889634f / sqrtf(static_cast<float>(d));
  cudaStream_t s = as_stream(stream);
  const int nq = ceil_div(max_len, attn::BM);
  int st;
  if (d % 128 == 0) {
    st = max_len <= 128 ? attn::launch_core<128, 128>(tm, seq_off, n_seq, 1, d, scale_log2e, ctx, s)
       : max_len <= 256 ? attn::launch_core<256, 128>(tm, seq_off, n_seq, nq, d, scale_log2e, ctx, s)
                        : attn::launch_core<512, 128>(tm, seq_off, n_seq, nq, d, scale_log2e, ctx, s);
  } else {
    st = max_len <= 128 ? attn::launch_core<128, 64>(tm, seq_off, n_seq, 1, d, scale_log2e, ctx, s)
       : max_len <= 256 ? attn::launch_core<256, 64>(tm, seq_off, n_seq, nq, d, scale_log2e, ctx, s)
                        : attn::launch_core<512, 64>(tm, seq_off, n_seq, nq, d, scale_log2e, ctx, s);
  }
  return st;
}
