// Expert FFN as a grouped bf16 GEMM on the 5th-gen tensor cores (sm_100a):
// TMA-fed, tcgen05.mma with the accumulator in TMEM, warp-specialised,
// persistent, with the bias/ReLU (GEMM1) and bias/alpha/unpermute/residual
// (GEMM2) epilogues fused. Replaces ref moe.py:235-262 (moe_apply), whose
// per-token gathered einsum is the reference's dominant cost.
//
// One launch = one GEMM over every (expert, 128-row tile, BN-col tile) of a
// layer. Rows are the permuted (token, rank) rows of sida_permute_hist, so
// each expert's rows are contiguous: tile (e, m) covers rows
// off[e] + 128m ... The B operand (W1^T or W2^T) is addressed in the HBM
// slot arena through a 3-D tensor map (k, n, slot) -- the residency engine
// moves experts between slots without rebuilding descriptors.
//
// CTA = 6 warps:  warp 0  TMA producer (one elected lane)
//                 warp 1  TMEM allocator + MMA issuer (one elected lane)
//                 warps 2-5 epilogue: TMEM -> registers -> global
// Pipelines: smem ring of kStages {A,B} stages (full/empty mbarriers),
// double-buffered TMEM accumulator (tmem_full/tmem_empty mbarriers) so the
// epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"

namespace sida {
namespace sm100 {

constexpr int BM = 128;       // UMMA M (cta_group::1), one TMEM lane per row
constexpr int BK = 64;        // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int UMMA_K = 16;    // K per tcgen05.mma for kind::f16
constexpr int kStages = 4;
constexpr int kThreads = 192;
constexpr int kMaxListed = 512;

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
  int stage;                   // 1: hidden = relu(acc + b1) bf16; 2: fp32 scatter epilogue
  uint16_t* hidden;            // stage 1 output (n_rows, ndim)
  const int32_t* row_map;      // stage 2
  const float* alpha;
  const float* resid;
  float* out;
  int32_t* err_flag;
};

// ---------------------------------------------------------------- PTX shims
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// K-major operand tile, 128-byte rows, SWIZZLE_128B, 8-row core groups 1024 B
// apart (canonical layout of cute::UMMA::make_umma_desc<Major::K>).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(1) << 16;            // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO
  d |= static_cast<uint64_t>(1) << 46;            // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: bf16 A/B, f32 D, both K-major, M=128.
template <int BN>
__device__ __forceinline__ constexpr uint32_t idesc_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ------------------------------------------------------------ tile schedule
struct TileInfo {
  int expert, row0, row_end, ncol0, slot;
};

__device__ __forceinline__ TileInfo decode_tile(int t, int n_ntiles, const int32_t* s_prefix,
                                                const int32_t* s_expert, int n_list,
                                                const GemmParams& p, int BN) {
  const int mt = t / n_ntiles, nt = t - mt * n_ntiles;
  int lo = 0, hi = n_list - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (s_prefix[mid] <= mt) lo = mid; else hi = mid - 1;
  }
  TileInfo ti;
  ti.expert = s_expert[lo];
  const int seg0 = p.off[ti.expert];
  ti.row0 = seg0 + (mt - s_prefix[lo]) * BM;
  ti.row_end = p.off[ti.expert + 1];
  ti.ncol0 = nt * BN;
  ti.slot = p.expert_slot[ti.expert];
  return ti;
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmParams p) {
  constexpr uint32_t kABytes = BM * BK * 2;
  constexpr uint32_t kBBytes = BN * BK * 2;
  constexpr uint32_t kTmemCols = 2 * BN;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tmem_full = bars + 2 * kStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  int32_t* s_prefix = reinterpret_cast<int32_t*>(s_tmem + 4);
  int32_t* s_expert = s_prefix + kMaxListed + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_list = p.expert_list ? p.n_list : p.num_experts;

  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < n_list; ++i) {
      const int e = p.expert_list ? p.expert_list[i] : i;
      s_expert[i] = e;
      s_prefix[i] = acc;
      acc += ceil_div(p.off[e + 1] - p.off[e], BM);
    }
    s_prefix[n_list] = acc;
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  const int n_ntiles = p.ndim / BN;
  const int total = s_prefix[n_list] * n_ntiles;
  const int n_kblocks = p.kdim / BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const TileInfo ti = decode_tile(t, n_ntiles, s_prefix, s_expert, n_list, p, BN);
        if (ti.slot < 0) continue;
        for (int kb = 0; kb < n_kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kABytes + kBBytes);
          tma_load_2d(sA + stage * kABytes, &tmA, kb * BK, ti.row0, &full[stage]);
          tma_load_3d(sB + stage * kBBytes, &tmB, kb * BK, ti.ncol0, ti.slot, &full[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16<BN>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const TileInfo ti = decode_tile(t, n_ntiles, s_prefix, s_expert, n_list, p, BN);
        if (ti.slot < 0) {
          atomicExch(p.err_flag, 1);
          continue;
        }
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < n_kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * kABytes);
          const uint32_t b0 = smem_u32(sB + stage * kBBytes);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            umma_bf16(d_tmem, sw128_desc(a0 + k * UMMA_K * 2), sw128_desc(b0 + k * UMMA_K * 2),
                      idesc, (kb | k) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tmem_full[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 == tile rows
    const int quarter = warp & 3;
    const int r_in_tile = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const TileInfo ti = decode_tile(t, n_ntiles, s_prefix, s_expert, n_list, p, BN);
      if (ti.slot < 0) continue;
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int row = ti.row0 + r_in_tile;
      const bool valid = row < ti.row_end;
      const uint16_t* bias = reinterpret_cast<const uint16_t*>(
          p.arena + static_cast<size_t>(ti.slot) * p.slot_stride + p.bias_off);
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN;
      float a_scale = 1.f;
      size_t orow = static_cast<size_t>(row);
      if (p.stage == 2 && valid) {
        if (p.alpha) a_scale = p.alpha[row];
        if (p.row_map) orow = static_cast<size_t>(p.row_map[row]);
      }
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(t_row + c * 32, v);
        const int col0 = ti.ncol0 + c * 32;
        if (!valid) continue;
        if (p.stage == 1) {
          uint4* dst = reinterpret_cast<uint4*>(p.hidden + orow * p.ndim + col0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              f[j] = fmaxf(__uint_as_float(v[q * 8 + j]) + bf16_to_f32(bias[col0 + q * 8 + j]), 0.f);
            uint4 o;
            o.x = pack_bf16x2(f[0], f[1]);
            o.y = pack_bf16x2(f[2], f[3]);
            o.z = pack_bf16x2(f[4], f[5]);
            o.w = pack_bf16x2(f[6], f[7]);
            dst[q] = o;
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(p.out + orow * p.ndim + col0);
          const float4* res = p.resid ? reinterpret_cast<const float4*>(p.resid + orow * p.ndim + col0)
                                      : nullptr;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4 o;
            o.x = (__uint_as_float(v[q * 4 + 0]) + bf16_to_f32(bias[col0 + q * 4 + 0])) * a_scale;
            o.y = (__uint_as_float(v[q * 4 + 1]) + bf16_to_f32(bias[col0 + q * 4 + 1])) * a_scale;
            o.z = (__uint_as_float(v[q * 4 + 2]) + bf16_to_f32(bias[col0 + q * 4 + 2])) * a_scale;
            o.w = (__uint_as_float(v[q * 4 + 3]) + bf16_to_f32(bias[col0 + q * 4 + 3])) * a_scale;
            if (res) {
              const float4 x = res[q];
              o.x = x.x + o.x; o.y = x.y + o.y; o.z = x.z + o.z; o.w = x.w + o.w;
            }
            dst[q] = o;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tmem_empty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

template <int BN>
constexpr size_t smem_bytes() {
  return 1024 + kStages * (BM * BK * 2 + BN * BK * 2) + (2 * kStages + 4) * 8 + 16 +
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

template <int BN>
static int launch_gemm(const void* a_base, const void* b_base, int n_slots, const GemmParams& p,
                       int n_listed, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    SIDA_CUDA(cudaFuncSetAttribute(grouped_gemm_kernel<BN>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_bytes<BN>()));
    configured = true;
  }
  CUtensorMap ta, tb;
  int st = make_map_2d(&ta, a_base, p.kdim, p.n_rows, BM);
  if (st) return st;
  st = make_map_3d(&tb, b_base, p.kdim, p.ndim, n_slots, p.slot_stride, BN);
  if (st) return st;
  const int max_tiles = (ceil_div(p.n_rows, BM) + n_listed) * (p.ndim / BN);
  const int grid = std::max(1, std::min(max_tiles, kNumSMs));
  grouped_gemm_kernel<BN><<<grid, kThreads, smem_bytes<BN>(), s>>>(ta, tb, p);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

static int dispatch_gemm(const void* a_base, const void* b_base, int n_slots, const GemmParams& p,
                         int n_listed, cudaStream_t s) {
  if (p.ndim % 256 == 0) return launch_gemm<256>(a_base, b_base, n_slots, p, n_listed, s);
  if (p.ndim % 128 == 0) return launch_gemm<128>(a_base, b_base, n_slots, p, n_listed, s);
  return launch_gemm<64>(a_base, b_base, n_slots, p, n_listed, s);
}

}  // namespace sm100
}  // namespace sida

using namespace sida;

extern "C" int sida_grouped_ffn_bf16(const uint16_t* x_perm, int n_rows, int d, int h,
                                     const int32_t* off, int num_experts,
                                     const int32_t* expert_slot, const int32_t* expert_list,
                                     int n_list, const void* arena, size_t slot_stride,
                                     int n_slots, const int32_t* row_map, const float* alpha,
                                     const float* resid, float* out, uint16_t* hidden,
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
  SIDA_REQUIRE(err_flag && out && hidden && x_perm && off && expert_slot && arena,
               SIDA_ERR_CONTRACT, "null pointer passed to sida_grouped_ffn_bf16");
  if (n_rows == 0 || listed == 0) return SIDA_OK;
  cudaStream_t s = as_stream(stream);
  const uint8_t* ar = static_cast<const uint8_t*>(arena);
  const size_t w2_off = (size_t)h * d * 2, b1_off = 2 * w2_off, b2_off = b1_off + (size_t)h * 2;

  sm100::GemmParams p1{};
  p1.n_rows = n_rows; p1.kdim = d; p1.ndim = h;
  p1.off = off; p1.num_experts = num_experts; p1.expert_slot = expert_slot;
  p1.expert_list = expert_list; p1.n_list = n_list;
  p1.arena = ar; p1.slot_stride = slot_stride; p1.bias_off = b1_off;
  p1.stage = 1; p1.hidden = hidden; p1.err_flag = err_flag;
  int st = sm100::dispatch_gemm(x_perm, ar, n_slots, p1, listed, s);
  if (st) return st;

  sm100::GemmParams p2 = p1;
  p2.kdim = h; p2.ndim = d; p2.bias_off = b2_off; p2.stage = 2;
  p2.row_map = row_map; p2.alpha = alpha; p2.resid = resid; p2.out = out;
  return sm100::dispatch_gemm(hidden, ar + w2_off, n_slots, p2, listed, s);
}
