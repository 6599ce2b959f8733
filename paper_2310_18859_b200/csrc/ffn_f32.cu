// fp32 FMA check path of the grouped expert FFN (SURVEY.md §2.1
// "ffn_fp32_check"): the same contraction as the bf16 tcgen05 kernel with
// float32 operands and reference-layout weights w1 (K,d,h), b1 (K,h),
// w2 (K,h,d), b2 (K,d) -- ref moe.py:235-262 -- so layer outputs can be held
// to rtol 1e-4 against the float64 oracle. Not on the throughput path.
#include <algorithm>

#include "common.cuh"

namespace sida {

constexpr int kF32Tile = 64, kF32K = 16, kF32Threads = 256;

// Expert segment -> tile-range bookkeeping shared by both GEMMs.
__device__ __forceinline__ void build_tile_prefix(const int32_t* off, int K, int32_t* s_prefix) {
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < K; ++e) {
      s_prefix[e] = acc;
      acc += ceil_div(off[e + 1] - off[e], kF32Tile);
    }
    s_prefix[K] = acc;
  }
  __syncthreads();
}

__device__ __forceinline__ int find_expert(const int32_t* s_prefix, int K, int mtile) {
  int lo = 0, hi = K - 1;
  while (lo < hi) {  // last e with prefix[e] <= mtile
    int mid = (lo + hi + 1) >> 1;
    if (s_prefix[mid] <= mtile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// GEMM over permuted rows. STAGE 1: hidden = relu(x W1_e + b1_e);
// STAGE 2: out[row_map[p]] = alpha[p] * (hidden W2_e + b2_e) (+ resid).
template <int STAGE>
__global__ void __launch_bounds__(kF32Threads)
ffn_f32_kernel(const float* __restrict__ A, int n_rows, int kdim, int ndim,
               const int32_t* __restrict__ off, int K, const float* __restrict__ W,
               const float* __restrict__ bias, const int32_t* __restrict__ row_map,
               const float* __restrict__ alpha, const float* __restrict__ resid,
               float* __restrict__ out) {
  extern __shared__ int32_t s_prefix[];
  __shared__ float sA[kF32K][kF32Tile + 4];
  __shared__ float sB[kF32K][kF32Tile];
  build_tile_prefix(off, K, s_prefix);
  const int n_tiles_n = ceil_div(ndim, kF32Tile);
  const int total = s_prefix[K] * n_tiles_n;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int mtile = t / n_tiles_n, ntile = t % n_tiles_n;
    const int e = find_expert(s_prefix, K, mtile);
    const int seg0 = off[e], seg1 = off[e + 1];
    const int row0 = seg0 + (mtile - s_prefix[e]) * kF32Tile;
    const int col0 = ntile * kF32Tile;
    const float* We = W + (size_t)e * kdim * ndim;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < kdim; k0 += kF32K) {
      for (int i = threadIdx.x; i < kF32K * kF32Tile; i += kF32Threads) {
        int r = i / kF32K, kk = i % kF32K;  // A tile: rows x K
        int gr = row0 + r, gk = k0 + kk;
        sA[kk][r] = (gr < seg1 && gk < kdim) ? A[(size_t)gr * kdim + gk] : 0.f;
        int kb = i / kF32Tile, c = i % kF32Tile;  // B tile: K x cols
        int gk2 = k0 + kb, gc = col0 + c;
        sB[kb][c] = (gk2 < kdim && gc < ndim) ? We[(size_t)gk2 * ndim + gc] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kF32K; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int p = row0 + ty * 4 + i;
      if (p >= seg1) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = col0 + tx * 4 + j;
        if (c >= ndim) continue;
        float v = acc[i][j] + bias[(size_t)e * ndim + c];
        if (STAGE == 1) {
          out[(size_t)p * ndim + c] = fmaxf(v, 0.f);
        } else {
          const size_t orow = row_map ? (size_t)row_map[p] : (size_t)p;
          if (alpha) v *= alpha[p];
          if (resid) v = resid[orow * ndim + c] + v;
          out[orow * ndim + c] = v;
        }
      }
    }
  }
}

}  // namespace sida

using namespace sida;

extern "C" int sida_grouped_ffn_f32(const float* x_perm, int n_rows, int d, int h,
                                    const int32_t* off, int num_experts, const float* w1,
                                    const float* b1, const float* w2, const float* b2,
                                    const int32_t* row_map, const float* alpha,
                                    const float* resid, float* out, float* hidden, void* stream) {
  SIDA_REQUIRE(n_rows >= 0 && d >= 1 && h >= 1 && num_experts >= 1 && num_experts <= 4096,
               SIDA_ERR_CONTRACT, "bad ffn dims");
  if (n_rows == 0) return SIDA_OK;
  cudaStream_t s = as_stream(stream);
  size_t smem = (num_experts + 1) * sizeof(int32_t);
  int max_tiles1 = (ceil_div(n_rows, kF32Tile) + num_experts) * ceil_div(h, kF32Tile);
  int max_tiles2 = (ceil_div(n_rows, kF32Tile) + num_experts) * ceil_div(d, kF32Tile);
  ffn_f32_kernel<1><<<std::min(max_tiles1, kNumSMs * 8), kF32Threads, smem, s>>>(
      x_perm, n_rows, d, h, off, num_experts, w1, b1, nullptr, nullptr, nullptr, hidden);
  SIDA_LAUNCH_CHECK();
  ffn_f32_kernel<2><<<std::min(max_tiles2, kNumSMs * 8), kF32Threads, smem, s>>>(
      hidden, n_rows, h, d, off, num_experts, w2, b2, row_map, alpha, resid, out);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}
