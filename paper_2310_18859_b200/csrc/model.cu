// The two thin ends of the MoE forward as kernels, so a serving step launches
// nothing but this library's kernels:
//   sida_embed          x[t] = tok_emb[tokens[t]] + pos_emb[t - seq_start(t)]
//                       (ref moe.py:206-218), fp32 residual stream plus its
//                       bf16 copy (the first QKV projection's input)
//   sida_pool_classify  logits[s] = mean_t x[t] @ wc over sequence s
//                       (ref moe.py:264-266)
// Both are HBM/latency-bound row kernels: one warp per token row (128-bit
// accesses) and one CTA per sequence.
#include <algorithm>

#include "common.cuh"

namespace sida {
namespace mdl {

// First token of the sequence holding token t (seq_off ascending, n_seq + 1).
__device__ __forceinline__ int seq_of(const int32_t* __restrict__ seq_off, int n_seq, int t) {
  int lo = 0, hi = n_seq - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(seq_off + mid) <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256)
embed_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ seq_off, int n_seq,
             int n_tokens, const uint16_t* __restrict__ tok_emb,
             const uint16_t* __restrict__ pos_emb, int d, float* __restrict__ x,
             uint16_t* __restrict__ xb) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int d8 = d >> 3;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_tokens; t += warps) {
    const int s = seq_of(seq_off, n_seq, t);
    const int pos = t - __ldg(seq_off + s);
    const uint4* te = reinterpret_cast<const uint4*>(tok_emb + (size_t)__ldg(tokens + t) * d);
    const uint4* pe = reinterpret_cast<const uint4*>(pos_emb + (size_t)pos * d);
    float4* xo = reinterpret_cast<float4*>(x + (size_t)t * d);
    uint4* bo = reinterpret_cast<uint4*>(xb + (size_t)t * d);
    for (int c = lane; c < d8; c += 32) {
      const uint4 a = __ldg(te + c), b = __ldg(pe + c);
      const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
      float f[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // bf16 + bf16 is exact in fp32
        f[2 * j] = __uint_as_float(aw[j] << 16) + __uint_as_float(bw[j] << 16);
        f[2 * j + 1] = __uint_as_float(aw[j] & 0xFFFF0000u) + __uint_as_float(bw[j] & 0xFFFF0000u);
      }
      xo[2 * c] = make_float4(f[0], f[1], f[2], f[3]);
      xo[2 * c + 1] = make_float4(f[4], f[5], f[6], f[7]);
      bo[c] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                         pack_bf16x2(f[6], f[7]));
    }
  }
}

// One CTA per sequence: column sums of its rows (thread = 4 columns, rows
// strided over the warps), then mean @ wc (thread per class, d-long dot).
__global__ void __launch_bounds__(256)
pool_classify_kernel(const float* __restrict__ x, const int32_t* __restrict__ seq_off, int d,
                     const float* __restrict__ wc, int n_cls, float* __restrict__ logits) {
  extern __shared__ float s_part[];  // [8 warps][d], then pooled [d]
  const int s = blockIdx.x;
  const int r0 = seq_off[s], r1 = seq_off[s + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* pooled = s_part + 8 * d;
  for (int c = lane * 4; c < d; c += 128) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = r0 + warp; r < r1; r += 8) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(x + (size_t)r * d + c));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    *reinterpret_cast<float4*>(s_part + warp * d + c) = acc;
  }
  __syncthreads();
  const float inv_n = 1.f / static_cast<float>(r1 - r0);
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_part[w * d + c];
    pooled[c] = t * inv_n;
  }
  __syncthreads();
  for (int k = warp; k < n_cls; k += 8) {
    float acc = 0.f;
    for (int c = lane; c < d; c += 32) acc = fmaf(pooled[c], __ldg(wc + (size_t)c * n_cls + k), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) logits[(size_t)s * n_cls + k] = acc;
  }
}

}  // namespace mdl
}  // namespace sida

using namespace sida;

extern "C" int sida_embed(const int32_t* tokens, const int32_t* seq_off, int n_seq, int n_tokens,
                          const uint16_t* tok_emb, const uint16_t* pos_emb, int d, float* x,
                          uint16_t* xb, void* stream) {
  SIDA_REQUIRE(d % 8 == 0, SIDA_ERR_UNSUPPORTED, "embed needs d %% 8 == 0 (d=%d)", d);
  SIDA_REQUIRE(n_seq >= 1 && n_tokens >= 0, SIDA_ERR_CONTRACT, "bad embed dims");
  SIDA_REQUIRE(tokens && seq_off && tok_emb && pos_emb && x && xb, SIDA_ERR_CONTRACT,
               "null pointer passed to sida_embed");
  if (n_tokens == 0) return SIDA_OK;
  const int blocks = std::min(ceil_div(n_tokens, 8), kNumSMs * 16);
  mdl::embed_kernel<<<blocks, 256, 0, as_stream(stream)>>>(tokens, seq_off, n_seq, n_tokens,
                                                           tok_emb, pos_emb, d, x, xb);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_pool_classify(const float* x, const int32_t* seq_off, int n_seq, int d,
                                  const float* wc, int n_cls, float* logits, void* stream) {
  SIDA_REQUIRE(d % 4 == 0 && d <= 8192, SIDA_ERR_UNSUPPORTED,
               "pool_classify needs d %% 4 == 0, d <= 8192 (d=%d)", d);
  SIDA_REQUIRE(n_seq >= 0 && n_cls >= 1, SIDA_ERR_CONTRACT, "bad pool dims");
  SIDA_REQUIRE(x && seq_off && wc && logits, SIDA_ERR_CONTRACT,
               "null pointer passed to sida_pool_classify");
  if (n_seq == 0) return SIDA_OK;
  const size_t smem = 9ull * d * sizeof(float);
  if (smem > 48 * 1024)
    SIDA_CUDA(cudaFuncSetAttribute(mdl::pool_classify_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  mdl::pool_classify_kernel<<<n_seq, 256, smem, as_stream(stream)>>>(x, seq_off, d, wc, n_cls,
                                                                     logits);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}
