// fp64 row kernels behind the reference's numeric API (ref numkit.py:28-93,
// moe.py:108-146): softmax, sparsemax and top-k over the rows of a matrix,
// the single-embedding router distribution (router_scores) and the
// single-token Eq. 1 expert mixture (moe_layer_forward). These are the
// drop-in's utility entry points, not the batched hot path (which fuses the
// same arithmetic into hash.cu / router.cu / ffn_sm100.cu), so each is one
// CTA per row with the row staged in shared memory.
//
// Exactness: sparsemax and top-k reproduce the reference bit for bit (same
// sort values, the sequential cumsum of np.cumsum, the same support test and
// tau formula; top-k = argsort(-z, kind="stable") ranks, ties to the lower
// index). softmax uses the GPU's exp and a tree sum, so it agrees with
// numpy's to a few ulp, not bit for bit.
#include <float.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace sida {
namespace nk {

constexpr int kThreads = 256;
constexpr int kMaxN = 8192;  // widest row (doubles in shared memory: 64 KB)

__device__ __forceinline__ double block_reduce(double v, bool is_max, double* s_red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, t) : v + t;
  }
  __syncthreads();
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? s_red[lane] : (is_max ? -DBL_MAX : 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmax(v, t) : v + t;
    }
    if (lane == 0) s_red[0] = v;
  }
  __syncthreads();
  return s_red[0];
}

// softmax(z) = exp(z - max z) / sum (ref numkit.py:28-33)
__global__ void __launch_bounds__(kThreads)
softmax_rows_kernel(const double* __restrict__ z, int n, double* __restrict__ out) {
  __shared__ double s_red[32];
  const double* row = z + (size_t)blockIdx.x * n;
  double* o = out + (size_t)blockIdx.x * n;
  double m = -DBL_MAX;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, row[i]);
  m = block_reduce(m, true, s_red);
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double e = exp(row[i] - m);
    o[i] = e;
    s += e;
  }
  s = block_reduce(s, false, s_red);
  for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = o[i] / s;
}

// Descending bitonic sort of s[0, np2) (np2 a power of two, padding -inf).
__device__ void bitonic_desc(double* s, int np2) {
  for (int k = 2; k <= np2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double a = s[i], b = s[ixj];
          const bool desc = (i & k) == 0;
          if (desc ? (a < b) : (a > b)) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Sparsemax closed form (ref numkit.py:42-60): sort descending, sequential
// cumsum, support = 1 + k z_(k) > cumsum_k (counted over every k, like
// np.count_nonzero), tau = (cumsum_{k_z} - 1) / k_z, out = max(z - tau, 0).
__global__ void __launch_bounds__(kThreads)
sparsemax_rows_kernel(const double* __restrict__ z, int n, int np2, double* __restrict__ out) {
  extern __shared__ double s_sort[];
  __shared__ double s_tau;
  const double* row = z + (size_t)blockIdx.x * n;
  for (int i = threadIdx.x; i < np2; i += blockDim.x) s_sort[i] = i < n ? row[i] : -INFINITY;
  __syncthreads();
  bitonic_desc(s_sort, np2);
  if (threadIdx.x == 0) {
    double cum = 0.0, cum_at = 0.0;
    int kz = 0;
    for (int k = 1; k <= n; ++k) {
      cum += s_sort[k - 1];
      if (1.0 + static_cast<double>(k) * s_sort[k - 1] > cum) ++kz;
    }
    // cums[k_z - 1]: recompute the prefix (the support may be non-contiguous
    // numerically; the reference indexes the cumsum at k_z - 1 regardless)
    for (int k = 0; k < kz; ++k) cum_at += s_sort[k];
    s_tau = (cum_at - 1.0) / static_cast<double>(kz);
  }
  __syncthreads();
  const double tau = s_tau;
  double* o = out + (size_t)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = fmax(row[i] - tau, 0.0);
}

// argsort(-z, kind="stable")[:k] (ref numkit.py:76-93): the rank of z_i is the
// number of larger entries plus the number of equal entries before it.
__global__ void __launch_bounds__(kThreads)
topk_rows_kernel(const double* __restrict__ z, int n, int k, int64_t* __restrict__ idx) {
  extern __shared__ double s_row[];
  const double* row = z + (size_t)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_row[i] = row[i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = s_row[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double u = s_row[j];
      rank += (u > v) || (u == v && j < i);
    }
    if (rank < k) idx[(size_t)blockIdx.x * k + rank] = i;
  }
}

// probs[r] = softmax(x[r] @ w_r) (ref moe.py:108-115 per embedding, batched
// over rows): one CTA per row, logits in shared memory.
__global__ void __launch_bounds__(kThreads)
router_scores_kernel(const double* __restrict__ x, int d, const double* __restrict__ w_r, int K,
                     double* __restrict__ probs) {
  extern __shared__ double s_logit[];
  __shared__ double s_red[32];
  const double* xr = x + (size_t)blockIdx.x * d;
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < d; ++i) acc = fma(xr[i], w_r[(size_t)i * K + e], acc);
    s_logit[e] = acc;
  }
  __syncthreads();
  double m = -DBL_MAX;
  for (int e = threadIdx.x; e < K; e += blockDim.x) m = fmax(m, s_logit[e]);
  m = block_reduce(m, true, s_red);
  double s = 0.0;
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    const double v = exp(s_logit[e] - m);
    s_logit[e] = v;
    s += v;
  }
  s = block_reduce(s, false, s_red);
  for (int e = threadIdx.x; e < K; e += blockDim.x)
    probs[(size_t)blockIdx.x * K + e] = s_logit[e] / s;
}

// Single-token Eq. 1 (ref moe.py:118-146), hidden half: one CTA per selected
// expert, hid[i] = relu(x @ w1_i + b1_i). Experts are packed in selection
// order: w1 (m, d, h), b1 (m, h).
__global__ void __launch_bounds__(kThreads)
moe_token_hidden_kernel(const double* __restrict__ x, const double* __restrict__ w1,
                        const double* __restrict__ b1, int d, int h, double* __restrict__ hid) {
  const int i = blockIdx.x;
  const double* w = w1 + (size_t)i * d * h;
  for (int j = threadIdx.x; j < h; j += blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < d; ++q) acc = fma(x[q], w[(size_t)q * h + j], acc);
    hid[(size_t)i * h + j] = fmax(acc + b1[(size_t)i * h + j], 0.0);
  }
}

// Output half: out[j] = sum_i alpha_i (hid_i @ w2_i + b2_i)[j], experts
// accumulated in selection order like the reference loop.
__global__ void __launch_bounds__(kThreads)
moe_token_out_kernel(const double* __restrict__ hid, const double* __restrict__ w2,
                     const double* __restrict__ b2, const double* __restrict__ alphas, int m,
                     int d, int h, double* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d; j += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < m; ++i) {
      const double* w = w2 + (size_t)i * h * d;
      const double* hi = hid + (size_t)i * h;
      double f = 0.0;
      for (int q = 0; q < h; ++q) f = fma(hi[q], w[(size_t)q * d + j], f);
      acc += alphas[i] * (f + b2[(size_t)i * d + j]);
    }
    out[j] = acc;
  }
}

}  // namespace nk
}  // namespace sida

using namespace sida;

extern "C" int sida_softmax_rows_f64(const double* z, int rows, int n, double* out, void* stream) {
  SIDA_REQUIRE(rows >= 0 && n >= 1 && z && out, SIDA_ERR_CONTRACT, "bad softmax rows=%d n=%d",
               rows, n);
  if (rows == 0) return SIDA_OK;
  nk::softmax_rows_kernel<<<rows, nk::kThreads, 0, as_stream(stream)>>>(z, n, out);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_sparsemax_rows_f64(const double* z, int rows, int n, double* out,
                                       void* stream) {
  SIDA_REQUIRE(rows >= 0 && n >= 1 && z && out, SIDA_ERR_CONTRACT, "bad sparsemax rows=%d n=%d",
               rows, n);
  SIDA_REQUIRE(n <= nk::kMaxN, SIDA_ERR_UNSUPPORTED, "sparsemax rows wider than %d", nk::kMaxN);
  if (rows == 0) return SIDA_OK;
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  const size_t smem = (size_t)np2 * sizeof(double);
  if (smem > 48 * 1024)
    SIDA_CUDA(cudaFuncSetAttribute(nk::sparsemax_rows_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  nk::sparsemax_rows_kernel<<<rows, nk::kThreads, smem, as_stream(stream)>>>(z, n, np2, out);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_topk_rows_f64(const double* z, int rows, int n, int k, int64_t* idx,
                                  void* stream) {
  SIDA_REQUIRE(rows >= 0 && n >= 1 && z && idx, SIDA_ERR_CONTRACT, "bad topk rows=%d n=%d", rows,
               n);
  SIDA_REQUIRE(k >= 1 && k <= n, SIDA_ERR_CONTRACT, "k=%d out of range for width-%d rows", k, n);
  SIDA_REQUIRE(n <= nk::kMaxN, SIDA_ERR_UNSUPPORTED, "top-k rows wider than %d", nk::kMaxN);
  if (rows == 0) return SIDA_OK;
  const size_t smem = (size_t)n * sizeof(double);
  if (smem > 48 * 1024)
    SIDA_CUDA(cudaFuncSetAttribute(nk::topk_rows_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  nk::topk_rows_kernel<<<rows, nk::kThreads, smem, as_stream(stream)>>>(z, n, k, idx);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_router_scores_f64(const double* x, int rows, int d, const double* w_r, int K,
                                      double* probs, void* stream) {
  SIDA_REQUIRE(rows >= 0 && d >= 1 && K >= 1 && x && w_r && probs, SIDA_ERR_CONTRACT,
               "bad router_scores rows=%d d=%d K=%d", rows, d, K);
  SIDA_REQUIRE(K <= nk::kMaxN, SIDA_ERR_UNSUPPORTED, "more than %d experts", nk::kMaxN);
  if (rows == 0) return SIDA_OK;
  const size_t smem = (size_t)K * sizeof(double);
  if (smem > 48 * 1024)
    SIDA_CUDA(cudaFuncSetAttribute(nk::router_scores_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  nk::router_scores_kernel<<<rows, nk::kThreads, smem, as_stream(stream)>>>(x, d, w_r, K, probs);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_moe_token_f64(const double* x, int m, const double* alphas, const double* w1,
                                  const double* b1, const double* w2, const double* b2, int d,
                                  int h, double* hidden, double* out, void* stream) {
  SIDA_REQUIRE(m >= 1 && d >= 1 && h >= 1, SIDA_ERR_CONTRACT, "bad moe token m=%d d=%d h=%d", m, d,
               h);
  SIDA_REQUIRE(x && alphas && w1 && b1 && w2 && b2 && hidden && out, SIDA_ERR_CONTRACT,
               "null pointer passed to sida_moe_token_f64");
  cudaStream_t s = as_stream(stream);
  nk::moe_token_hidden_kernel<<<m, nk::kThreads, 0, s>>>(x, w1, b1, d, h, hidden);
  SIDA_LAUNCH_CHECK();
  nk::moe_token_out_kernel<<<std::max(1, ceil_div(d, nk::kThreads)), nk::kThreads, 0, s>>>(
      hidden, w2, b2, alphas, m, d, h, out);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}
