// Token permute + histogram, every MoE layer of a
// batch in one pass, plus the bf16 row gather.
//
// The reference never permutes: moe_apply gathers w1[ids] per token
// (ref moe.py:253-256). The GPU path groups the (token, rank) rows of each
// layer by expert with a stable counting sort whose output is bit-identical
// to np.argsort(ids[l].reshape(-1), kind="stable") (oracle/permute.py):
//
//   hist_tiles : per (layer, tile of kTileRows rows) smem histogram
//   scan       : per layer, exclusive scan over (expert-major, tile-minor)
//                -> off[l] and each (expert, tile) base position
//   scatter    : per tile, rows visited in order; the within-warp stable rank
//                comes from __match_any_sync + popc (warp-shuffle prefix),
//                the cross-warp prefix from a per-chunk smem count table.
//
// Since SiDA's hash table holds every layer's ids before inference starts
// (ref pipeline.py:208-215), all L layers are permuted in one launch on the
// hash stream; only the x-row gather waits for each layer's input.
#include <algorithm>

#include "common.cuh"

namespace sida {

constexpr int kTileRows = 4096;
constexpr int kPermThreads = 256;
constexpr int kPermWarps = kPermThreads / 32;
constexpr int kMaxExperts = 1024;

__global__ void __launch_bounds__(kPermThreads)
hist_tiles_kernel(const int32_t* __restrict__ ids, int n_rows, int K, int n_tiles,
                  int32_t* __restrict__ tile_counts, int32_t* __restrict__ err) {
  extern __shared__ int32_t s_hist[];
  const int layer = blockIdx.y, tile = blockIdx.x;
  for (int e = threadIdx.x; e < K; e += blockDim.x) s_hist[e] = 0;
  __syncthreads();
  const int32_t* row_ids = ids + (size_t)layer * n_rows;
  const int r0 = tile * kTileRows, r1 = min(n_rows, r0 + kTileRows);
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    int e = row_ids[r];
    if (e < 0 || e >= K) {
      atomicExch(err, 1);
      continue;
    }
    atomicAdd(&s_hist[e], 1);
  }
  __syncthreads();
  int32_t* tc = tile_counts + (size_t)layer * K * n_tiles;
  for (int e = threadIdx.x; e < K; e += blockDim.x) tc[(size_t)e * n_tiles + tile] = s_hist[e];
}

// One block per layer: exclusive scan of tile_counts in (expert, tile) order.
__global__ void __launch_bounds__(1024)
scan_kernel(const int32_t* __restrict__ tile_counts, int K, int n_tiles,
            int32_t* __restrict__ tile_base, int32_t* __restrict__ hist, int32_t* __restrict__ off) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  const int layer = blockIdx.x;
  const size_t n = (size_t)K * n_tiles;
  const int32_t* tc = tile_counts + (size_t)layer * n;
  int32_t* tb = tile_base + (size_t)layer * n;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (size_t base = 0; base < n; base += blockDim.x) {
    size_t i = base + threadIdx.x;
    int v = i < n ? tc[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      s_warp[lane] = wi - w;  // exclusive per-warp prefix
    }
    __syncthreads();
    const int carry = s_carry;
    if (i < n) tb[i] = carry + s_warp[warp] + incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = carry + s_warp[warp] + incl;
    __syncthreads();
  }
  // hist / off from the per-expert sums
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    int s = 0;
    for (int t = 0; t < n_tiles; ++t) s += tc[(size_t)e * n_tiles + t];
    hist[(size_t)layer * K + e] = s;
    off[(size_t)layer * (K + 1) + e] = tb[(size_t)e * n_tiles];
  }
  if (threadIdx.x == 0) off[(size_t)layer * (K + 1) + K] = s_carry;
}

__global__ void __launch_bounds__(kPermThreads)
scatter_kernel(const int32_t* __restrict__ ids, int n_rows, int K, int n_tiles,
               const int32_t* __restrict__ tile_base, const float* __restrict__ alpha_rows,
               int32_t* __restrict__ perm, int32_t* __restrict__ inv,
               float* __restrict__ alpha_perm) {
  extern __shared__ int32_t smem[];
  int32_t* s_run = smem;                    // [K] running count of this tile
  int32_t* s_warp = smem + K;               // [kPermWarps][K] counts of this chunk
  const int layer = blockIdx.y, tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t* row_ids = ids + (size_t)layer * n_rows;
  const int32_t* tb = tile_base + (size_t)layer * K * n_tiles;
  int32_t* lperm = perm + (size_t)layer * n_rows;
  int32_t* linv = inv + (size_t)layer * n_rows;
  for (int e = threadIdx.x; e < K; e += blockDim.x) s_run[e] = tb[(size_t)e * n_tiles + tile];
  for (int i = threadIdx.x; i < kPermWarps * K; i += blockDim.x) s_warp[i] = 0;
  __syncthreads();
  const unsigned lt_mask = (1u << lane) - 1u;
  const int r0 = tile * kTileRows, r1 = min(n_rows, r0 + kTileRows);
  for (int c0 = r0; c0 < r1; c0 += kPermThreads) {
    const int r = c0 + threadIdx.x;
    const bool valid = r < r1;
    int e = valid ? row_ids[r] : -1;
    if (valid && (e < 0 || e >= K)) e = -1;  // counted as error by hist pass
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(peers & lt_mask);
    const bool leader = (peers & lt_mask) == 0;
    if (e >= 0 && leader) s_warp[warp * K + e] = __popc(peers);
    __syncthreads();
    if (e >= 0) {
      int pos = s_run[e] + rank;
      for (int w = 0; w < warp; ++w) pos += s_warp[w * K + e];
      lperm[pos] = r;
      linv[r] = pos;
      if (alpha_perm) alpha_perm[(size_t)layer * n_rows + pos] = alpha_rows[(size_t)layer * n_rows + r];
    }
    __syncthreads();
    for (int x = threadIdx.x; x < K; x += blockDim.x) {
      int s = 0;
#pragma unroll
      for (int w = 0; w < kPermWarps; ++w) {
        s += s_warp[w * K + x];
        s_warp[w * K + x] = 0;
      }
      s_run[x] += s;
    }
    __syncthreads();
  }
}

// x_perm[p] = bf16(x[perm[p] / k]); one warp per row, 128-bit loads/stores.
__global__ void __launch_bounds__(256)
gather_rows_kernel(const float* __restrict__ x, const int32_t* __restrict__ perm, int n_rows, int k,
                   int d, uint16_t* __restrict__ x_perm) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int d8 = d >> 3;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n_rows; p += warps) {
    const int tok = perm[p] / k;
    const float4* src = reinterpret_cast<const float4*>(x + (size_t)tok * d);
    uint4* dst = reinterpret_cast<uint4*>(x_perm + (size_t)p * d);
    for (int c = lane; c < d8; c += 32) {
      float4 a = __ldg(src + 2 * c), b = __ldg(src + 2 * c + 1);
      uint4 o;
      o.x = pack_bf16x2(a.x, a.y);
      o.y = pack_bf16x2(a.z, a.w);
      o.z = pack_bf16x2(b.x, b.y);
      o.w = pack_bf16x2(b.z, b.w);
      dst[c] = o;
    }
  }
}

}  // namespace sida

using namespace sida;

static inline int perm_tiles(int n_rows) { return std::max(1, ceil_div(n_rows, kTileRows)); }

extern "C" size_t sida_permute_workspace_bytes(int n_layers, int n_rows, int num_experts) {
  size_t n = (size_t)n_layers * num_experts * perm_tiles(n_rows);
  return align_up(2 * n * sizeof(int32_t), 256) + 256;
}

extern "C" int sida_permute_hist(const int32_t* ids, int n_layers, int n_rows, int num_experts,
                                 const float* alpha_rows, int32_t* hist, int32_t* off,
                                 int32_t* perm, int32_t* inv, float* alpha_perm, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  SIDA_REQUIRE(n_layers >= 1 && n_rows >= 0 && num_experts >= 1, SIDA_ERR_CONTRACT,
               "bad permute dims L=%d rows=%d K=%d", n_layers, n_rows, num_experts);
  SIDA_REQUIRE(num_experts <= kMaxExperts, SIDA_ERR_UNSUPPORTED, "K=%d > %d", num_experts,
               kMaxExperts);
  SIDA_REQUIRE(workspace_bytes >= sida_permute_workspace_bytes(n_layers, n_rows, num_experts),
               SIDA_ERR_CONTRACT, "permute workspace too small");
  SIDA_REQUIRE(!alpha_perm || alpha_rows, SIDA_ERR_CONTRACT, "alpha_perm needs alpha_rows");
  cudaStream_t s = as_stream(stream);
  const int n_tiles = perm_tiles(n_rows);
  size_t n = (size_t)n_layers * num_experts * n_tiles;
  int32_t* tile_counts = static_cast<int32_t*>(workspace);
  int32_t* tile_base = tile_counts + n;
  int32_t* err = reinterpret_cast<int32_t*>(static_cast<char*>(workspace) +
                                            align_up(2 * n * sizeof(int32_t), 256));
  SIDA_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), s));
  dim3 grid(n_tiles, n_layers);
  hist_tiles_kernel<<<grid, kPermThreads, num_experts * sizeof(int32_t), s>>>(
      ids, n_rows, num_experts, n_tiles, tile_counts, err);
  SIDA_LAUNCH_CHECK();
  scan_kernel<<<n_layers, 1024, 0, s>>>(tile_counts, num_experts, n_tiles, tile_base, hist, off);
  SIDA_LAUNCH_CHECK();
  if (n_rows > 0) {
    size_t smem = (size_t)(1 + kPermWarps) * num_experts * sizeof(int32_t);
    scatter_kernel<<<grid, kPermThreads, smem, s>>>(ids, n_rows, num_experts, n_tiles, tile_base,
                                                    alpha_rows, perm, inv, alpha_perm);
    SIDA_LAUNCH_CHECK();
  }
  return SIDA_OK;
}

// dst[p] = src[idx[p]] for bf16 rows (16-byte vectors): the expert-parallel
// regroup of received rows into local expert-major order.
__global__ void __launch_bounds__(256)
gather_bf16_rows_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ idx, int n_rows,
                        int d8, uint4* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n_rows; p += warps) {
    const uint4* s = src + (size_t)idx[p] * d8;
    uint4* o = dst + (size_t)p * d8;
    for (int c = lane; c < d8; c += 32) o[c] = __ldg(s + c);
  }
}

// out[t] = resid[t] + sum_{r<k} alpha_perm[inv[t*k+r]] * y_perm[inv[t*k+r]] (ranks in
// order, ref moe.py:252-262): the combine of expert-parallel outputs that
// come back in the source rank's permuted row order. One warp per token.
__global__ void __launch_bounds__(256)
unpermute_combine_kernel(const uint16_t* __restrict__ y_perm, const int32_t* __restrict__ inv,
                         const float* __restrict__ alpha_perm, const float* __restrict__ resid,
                         int n_tokens, int k, int d, float* __restrict__ out,
                         uint16_t* __restrict__ out_bf16) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_tokens; t += warps) {
    for (int c = lane * 4; c < d; c += 128) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int r = 0; r < k; ++r) {
        const int p = inv[(size_t)t * k + r];
        const float a = alpha_perm[p];
        const uint2 raw = *reinterpret_cast<const uint2*>(y_perm + (size_t)p * d + c);
        acc.x += a * bf16_to_f32(static_cast<uint16_t>(raw.x & 0xFFFF));
        acc.y += a * bf16_to_f32(static_cast<uint16_t>(raw.x >> 16));
        acc.z += a * bf16_to_f32(static_cast<uint16_t>(raw.y & 0xFFFF));
        acc.w += a * bf16_to_f32(static_cast<uint16_t>(raw.y >> 16));
      }
      const float4 x = *reinterpret_cast<const float4*>(resid + (size_t)t * d + c);
      const float4 o = make_float4(x.x + acc.x, x.y + acc.y, x.z + acc.z, x.w + acc.w);
      *reinterpret_cast<float4*>(out + (size_t)t * d + c) = o;
      if (out_bf16)
        *reinterpret_cast<uint2*>(out_bf16 + (size_t)t * d + c) =
            make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
    }
  }
}

extern "C" int sida_gather_bf16_rows(const uint16_t* src, const int32_t* idx, int n_rows, int d,
                                     uint16_t* dst, void* stream) {
  SIDA_REQUIRE(d % 8 == 0, SIDA_ERR_UNSUPPORTED, "bf16 gather needs d %% 8 == 0 (d=%d)", d);
  if (n_rows == 0) return SIDA_OK;
  const int blocks = std::min(ceil_div(n_rows, 8), kNumSMs * 16);
  gather_bf16_rows_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(src), idx, n_rows, d / 8, reinterpret_cast<uint4*>(dst));
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_unpermute_combine(const uint16_t* y_perm, const int32_t* inv,
                                      const float* alpha_perm, const float* resid, int n_tokens,
                                      int k, int d, float* out, uint16_t* out_bf16, void* stream) {
  SIDA_REQUIRE(d % 4 == 0 && k >= 1, SIDA_ERR_UNSUPPORTED, "combine needs d %% 4 == 0 (d=%d)", d);
  SIDA_REQUIRE(y_perm && inv && alpha_perm && resid && out, SIDA_ERR_CONTRACT,
               "null pointer passed to sida_unpermute_combine");
  if (n_tokens == 0) return SIDA_OK;
  const int blocks = std::min(ceil_div(n_tokens, 8), kNumSMs * 16);
  unpermute_combine_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      y_perm, inv, alpha_perm, resid, n_tokens, k, d, out, out_bf16);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_gather_rows_bf16(const float* x, const int32_t* perm, int n_rows, int k, int d,
                                     uint16_t* x_perm, void* stream) {
  SIDA_REQUIRE(d % 8 == 0, SIDA_ERR_UNSUPPORTED, "gather needs d %% 8 == 0 (d=%d)", d);
  SIDA_REQUIRE(k >= 1, SIDA_ERR_CONTRACT, "k must be >= 1");
  if (n_rows == 0) return SIDA_OK;
  int blocks = std::min(ceil_div(n_rows, 8), kNumSMs * 16);
  gather_rows_kernel<<<blocks, 256, 0, as_stream(stream)>>>(x, perm, n_rows, k, d, x_perm);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}
