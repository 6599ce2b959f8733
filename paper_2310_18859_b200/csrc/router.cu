// Router-mode expert selection (the teacher path): z = x W_r, softmax over
// the K experts, top-k with the reference's tie rule, fused in one kernel.
// Replaces ref moe.py:296-301 (`softmax(x @ w_r)`, `topk_rows(probs, k)`,
// `take_along_axis`), numkit.py:28-33 / :87-93, used by router-mode
// `model_forward`, `OracleHasher` (ref predictor.py:413-426) and
// `serve_standard` (ref pipeline.py:370-377).
//
// CTA = 256 threads = 32 tokens x 8 lanes. Lane q of a token owns experts
// q, q+8, q+16, ... (MAXJ per thread), so the d-loop reads each x value once
// per token from shared memory (broadcast across the 8 lanes) and the W_r
// chunk once per CTA. z accumulates in fp32 FMAs over fp32 activations and
// the bf16-valued router weights; the softmax and the top-k comparisons run
// in fp64 (the reference's arithmetic type) on those z.
//
// top-k order = np.argsort(-p, kind="stable")[:k]: descending probability,
// equal probabilities to the lower expert index.
#include <math.h>

#include "common.cuh"

namespace sida {
namespace router {

constexpr int kTok = 32;   // tokens per CTA
constexpr int kLanes = 8;  // threads per token
constexpr int kDC = 32;    // d-chunk staged in shared memory
constexpr int kMaxK = 256;

template <int MAXJ>
__global__ void __launch_bounds__(kTok* kLanes)
router_topk_kernel(const float* __restrict__ x, int n, int d, const float* __restrict__ w, int K,
                   int ktop, float* __restrict__ probs, int32_t* __restrict__ sel,
                   double* __restrict__ alpha, float* __restrict__ alpha_f32) {
  __shared__ float xs[kTok][kDC + 1];
  extern __shared__ float ws[];  // [kDC][K]
  const int tid = threadIdx.x;
  const int tl = tid / kLanes, q = tid % kLanes;
  const int tok0 = blockIdx.x * kTok;
  const int tok = tok0 + tl;

  float acc[MAXJ];
#pragma unroll
  for (int j = 0; j < MAXJ; ++j) acc[j] = 0.f;

  for (int d0 = 0; d0 < d; d0 += kDC) {
    const int dc = min(kDC, d - d0);
    for (int i = tid; i < kTok * kDC; i += blockDim.x) {
      const int r = i / kDC, c = i % kDC;
      xs[r][c] = (tok0 + r < n && c < dc) ? x[static_cast<size_t>(tok0 + r) * d + d0 + c] : 0.f;
    }
    for (int i = tid; i < dc * K; i += blockDim.x) ws[i] = w[static_cast<size_t>(d0) * K + i];
    __syncthreads();
    for (int c = 0; c < dc; ++c) {
      const float xv = xs[tl][c];
      const float* wr = ws + c * K;
#pragma unroll
      for (int j = 0; j < MAXJ; ++j) {
        const int e = q + kLanes * j;
        if (e < K) acc[j] = fmaf(xv, wr[e], acc[j]);
      }
    }
    __syncthreads();
  }
  const bool valid = tok < n;  // (no early exit: the 8-lane shuffles below need the warp)

  // softmax over the token's K logits (fp64), spread over its 8 lanes
  double m = -INFINITY;
#pragma unroll
  for (int j = 0; j < MAXJ; ++j)
    if (q + kLanes * j < K) m = fmax(m, static_cast<double>(acc[j]));
#pragma unroll
  for (int o = 4; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o, kLanes));
  double p[MAXJ];
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < MAXJ; ++j) {
    p[j] = q + kLanes * j < K ? exp(static_cast<double>(acc[j]) - m) : 0.0;
    s += p[j];
  }
#pragma unroll
  for (int o = 4; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, kLanes);
#pragma unroll
  for (int j = 0; j < MAXJ; ++j) {
    p[j] /= s;
    const int e = q + kLanes * j;
    if (probs && valid && e < K) probs[static_cast<size_t>(tok) * K + e] = static_cast<float>(p[j]);
  }

  // top-k: k rounds of a (prob desc, index asc) argmax over the 8 lanes
  uint32_t taken = 0;
  for (int r = 0; r < ktop; ++r) {
    double bp = -1.0;
    int be = 0x7fffffff, bj = -1;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int e = q + kLanes * j;
      if (e < K && !(taken >> j & 1u) && p[j] > bp) {  // ascending j: first max = lowest e
        bp = p[j];
        be = e;
        bj = j;
      }
    }
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      const double op = __shfl_xor_sync(0xffffffffu, bp, o, kLanes);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o, kLanes);
      if (op > bp || (op == bp && oe < be)) {
        bp = op;
        be = oe;
      }
    }
    if (bj >= 0 && q + kLanes * bj == be) taken |= 1u << bj;
    if (q == 0 && valid) {
      const size_t at = static_cast<size_t>(tok) * ktop + r;
      sel[at] = be;
      alpha[at] = bp;
      if (alpha_f32) alpha_f32[at] = static_cast<float>(bp);
    }
  }
}

template <int MAXJ>
static int launch(const float* x, int n, int d, const float* w, int K, int ktop, float* probs,
                  int32_t* sel, double* alpha, float* alpha_f32, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(kDC) * K * sizeof(float);
  router_topk_kernel<MAXJ><<<ceil_div(n, kTok), kTok * kLanes, smem, s>>>(
      x, n, d, w, K, ktop, probs, sel, alpha, alpha_f32);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

}  // namespace router
}  // namespace sida

using namespace sida;

extern "C" int sida_router_topk(const float* x, int n_tokens, int d, const float* w_r,
                                int num_experts, int k, float* probs, int32_t* ids,
                                double* alpha, float* alpha_f32, void* stream) {
  SIDA_REQUIRE(n_tokens >= 0 && d >= 1, SIDA_ERR_CONTRACT, "bad router dims n=%d d=%d", n_tokens,
               d);
  SIDA_REQUIRE(num_experts >= 1 && num_experts <= router::kMaxK, SIDA_ERR_UNSUPPORTED,
               "router supports 1..%d experts (got %d)", router::kMaxK, num_experts);
  SIDA_REQUIRE(k >= 1 && k <= num_experts, SIDA_ERR_CONTRACT,
               "k=%d out of range for width-%d rows", k, num_experts);
  SIDA_REQUIRE(x && w_r && ids && alpha, SIDA_ERR_CONTRACT, "null pointer passed to sida_router_topk");
  if (n_tokens == 0) return SIDA_OK;
  cudaStream_t s = as_stream(stream);
  const int per = ceil_div(num_experts, router::kLanes);
#define SIDA_ROUTER(J) \
  return router::launch<J>(x, n_tokens, d, w_r, num_experts, k, probs, ids, alpha, alpha_f32, s)
  if (per <= 1) SIDA_ROUTER(1);
  if (per <= 2) SIDA_ROUTER(2);
  if (per <= 4) SIDA_ROUTER(4);
  if (per <= 8) SIDA_ROUTER(8);
  if (per <= 16) SIDA_ROUTER(16);
  SIDA_ROUTER(32);
#undef SIDA_ROUTER
}
