// Token permute + histogram, every MoE layer of a
// batch in one launch chain, plus the bf16 row gather.
//
// The reference never permutes: moe_apply gathers w1[ids] per token
// (ref moe.py:253-256). The GPU path groups the (token, rank) rows of each
// layer by expert with a stable counting sort whose output is bit-identical
// to np.argsort(ids[l].reshape(-1), kind="stable") (oracle/permute.py).
// Rows are cut into tiles of TILE rows (1024..8192, chosen so that L x tiles
// covers >= 2 CTAs per SM); one CTA of 256 threads per (layer, tile):
//
//   hist_tiles : 128-bit id loads into shared memory, warp-aggregated
//                (__match_any_sync) shared histogram -> counts[l][tile][e]
//   scan       : per layer, one thread per expert: totals over tiles
//                (coalesced across experts), block exclusive scan -> off,
//                then each (tile, expert) base position
//   scatter    : the tile's ids staged again in shared memory; each warp
//                walks its contiguous rows in order and takes the in-warp
//                stable rank from __match_any_sync + popc, per-warp running
//                counts give the cross-warp prefix; inv is written row-ordered
//                (coalesced), then perm / alpha_perm are written from a
//                shared-memory copy of the tile in sorted order, so every
//                (tile, expert) run is a contiguous store.
//
// Since SiDA's hash table holds every layer's ids before inference starts
// (ref pipeline.py:208-215), all L layers are permuted in one chain on the
// hash stream; only the x-row gather waits for each layer's input.
#include <algorithm>

#include "common.cuh"

namespace sida {

constexpr int kPermThreads = 256;
constexpr int kPermWarps = kPermThreads / 32;
constexpr int kMaxExperts = 1024;

// Tile rows for (rows, layers): >= 2 CTAs per SM when the batch allows it.
static inline int perm_tile(int n_rows, int n_layers) {
  const long long want = (long long)n_rows * std::max(n_layers, 1) / (2 * kNumSMs);
  int t = 1024;
  while (t < 8192 && 2ll * t <= want) t *= 2;
  return t;
}

static inline int perm_tiles(int n_rows, int tile) { return std::max(1, ceil_div(n_rows, tile)); }

// Stage ids[r0, r1) of one layer into shared memory (128-bit loads when aligned).
__device__ __forceinline__ void stage_ids(const int32_t* __restrict__ row_ids, int r0, int r1,
                                          int32_t* __restrict__ s_ids) {
  const int n = r1 - r0;
  const int32_t* src = row_ids + r0;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int n4 = n >> 2;
    const int4* s4 = reinterpret_cast<const int4*>(src);
    for (int i = threadIdx.x; i < n4; i += blockDim.x)
      reinterpret_cast<int4*>(s_ids)[i] = __ldg(s4 + i);
    for (int i = (n4 << 2) + threadIdx.x; i < n; i += blockDim.x) s_ids[i] = __ldg(src + i);
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_ids[i] = __ldg(src + i);
  }
}

template <int TILE>
__global__ void __launch_bounds__(kPermThreads)
hist_tiles_kernel(const int32_t* __restrict__ ids, int n_rows, int K, int n_tiles,
                  int32_t* __restrict__ counts, int32_t* __restrict__ err) {
  __shared__ int32_t s_ids[TILE];
  extern __shared__ int32_t s_hist[];  // [K]
  const int layer = blockIdx.y, tile = blockIdx.x;
  const int lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int e = threadIdx.x; e < K; e += blockDim.x) s_hist[e] = 0;
  const int r0 = tile * TILE, r1 = min(n_rows, r0 + TILE);
  stage_ids(ids + (size_t)layer * n_rows, r0, r1, s_ids);
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  bool bad = false;
  for (int i = threadIdx.x; i < TILE; i += blockDim.x) {  // uniform trip count: full warps
    int e = i < r1 - r0 ? s_ids[i] : -1;
    if (i < r1 - r0 && (e < 0 || e >= K)) { bad = true; e = -1; }
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    if (e >= 0 && (peers & lt) == 0) atomicAdd(&s_hist[e], __popc(peers));
  }
  if (bad) atomicExch(err, 1);
  __syncthreads();
  int32_t* c = counts + ((size_t)layer * n_tiles + tile) * K;
  for (int e = threadIdx.x; e < K; e += blockDim.x) c[e] = s_hist[e];
}

template <int TILE>
__global__ void __launch_bounds__(kPermThreads, 2)
scatter_kernel(const int32_t* __restrict__ ids, int n_rows, int K, int n_tiles,
               const int32_t* __restrict__ counts, const float* __restrict__ alpha_rows,
               int32_t* __restrict__ perm, int32_t* __restrict__ inv,
               float* __restrict__ alpha_perm, int32_t* __restrict__ hist,
               int32_t* __restrict__ off) {
  constexpr int R = TILE / kPermWarps;  // contiguous rows per warp
  constexpr int NR = R / 32;            // rounds per warp
  extern __shared__ int32_t smem[];
  int32_t* s_ids = smem;                        // [TILE] ids, then sorted rows
  int32_t* s_ord = s_ids + TILE;                // [TILE] tile row of sorted position q
  int32_t* s_cnt = s_ord + TILE;                // [warps][K] counts -> warp prefix
  int32_t* s_tbase = s_cnt + kPermWarps * K;    // [K] global base of (tile, e)
  int32_t* s_texc = s_tbase + K;                // [K + 1] tile-local exclusive prefix
  const int layer = blockIdx.y, tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = tile * TILE, r1 = min(n_rows, r0 + TILE), n = r1 - r0;
  for (int i = threadIdx.x; i < kPermWarps * K; i += blockDim.x) s_cnt[i] = 0;
  stage_ids(ids + (size_t)layer * n_rows, r0, r1, s_ids);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // hist_tiles' counts are complete
  // this tile's base positions from the layer's (tile, expert) count matrix
  // (written by hist_tiles; n_tiles x K ints read from L2): per expert the
  // total and the count in earlier tiles, then an exclusive scan of the
  // totals over experts; tile 0 also publishes hist / off
  const int32_t* cl = counts + (size_t)layer * n_tiles * K;
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    int tot = 0, pre = 0;
    for (int t = 0; t < n_tiles; ++t) {
      const int c = __ldg(cl + (size_t)t * K + e);
      tot += c;
      pre += t < tile ? c : 0;
    }
    s_texc[e] = tot;
    s_tbase[e] = pre;
  }
  __syncthreads();
  if (warp == 0) {
    int carry = 0;
    for (int b = 0; b < K; b += 32) {
      const int e = b + lane;
      const int v = e < K ? s_texc[e] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (e < K) {
        s_tbase[e] += carry + incl - v;
        if (tile == 0) {
          hist[(size_t)layer * K + e] = v;
          off[(size_t)layer * (K + 1) + e] = carry + incl - v;
        }
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tile == 0 && lane == 0) off[(size_t)layer * (K + 1) + K] = carry;
  }
  __syncthreads();

  // pass 1: in-order stable local ranks, per warp over its R rows
  const unsigned lt = (1u << lane) - 1u;
  int32_t* my_cnt = s_cnt + warp * K;
  int loc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int i = warp * R + j * 32 + lane;
    int e = i < n ? s_ids[i] : -1;
    if (e >= K) e = -1;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    int base = 0;
    if (e >= 0) base = my_cnt[e];
    __syncwarp();
    if (e >= 0 && (peers & lt) == 0) my_cnt[e] = base + __popc(peers);
    __syncwarp();
    loc[j] = base + __popc(peers & lt);
  }
  __syncthreads();

  // warp prefix per expert (in place) and the tile's per-expert totals
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < kPermWarps; ++w) {
      const int c = s_cnt[w * K + e];
      s_cnt[w * K + e] = run;
      run += c;
    }
    s_texc[e] = run;  // total; scanned below
  }
  __syncthreads();
  // exclusive scan of the totals over experts (one warp, K <= 1024)
  if (warp == 0) {
    int carry = 0;
    for (int b = 0; b < K; b += 32) {
      const int e = b + lane;
      const int v = e < K ? s_texc[e] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (e < K) s_texc[e] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_texc[K] = carry;
  }
  __syncthreads();

  // pass 2: positions; inv row-ordered, sorted order staged in shared memory
  int32_t* linv = inv + (size_t)layer * n_rows;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int i = warp * R + j * 32 + lane;
    int e = i < n ? s_ids[i] : -1;
    if (e >= K) e = -1;
    if (e >= 0) {
      const int within = s_cnt[warp * K + e] + loc[j];
      linv[r0 + i] = s_tbase[e] + within;
      s_ord[s_texc[e] + within] = i;
    } else if (i < n) {
      linv[r0 + i] = -1;
    }
  }
  __syncthreads();
  const int n_valid = s_texc[K];
  int32_t* lperm = perm + (size_t)layer * n_rows;
  const float* la = alpha_rows ? alpha_rows + (size_t)layer * n_rows + r0 : nullptr;
  float* lap = alpha_perm ? alpha_perm + (size_t)layer * n_rows : nullptr;
  for (int q = threadIdx.x; q < n_valid; q += blockDim.x) {
    const int i = s_ord[q];
    const int e = s_ids[i];
    const int pos = s_tbase[e] + (q - s_texc[e]);
    lperm[pos] = r0 + i;
    if (lap) lap[pos] = la[i];
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

extern "C" size_t sida_permute_workspace_bytes(int n_layers, int n_rows, int num_experts) {
  const int tile = perm_tile(n_rows, n_layers);
  size_t n = (size_t)n_layers * num_experts * perm_tiles(n_rows, tile);
  return align_up(2 * n * sizeof(int32_t), 256);
}

template <int TILE>
static int permute_launch(const int32_t* ids, int n_layers, int n_rows, int K, const float* alpha_rows,
                          int32_t* hist, int32_t* off, int32_t* perm, int32_t* inv,
                          float* alpha_perm, int32_t* counts, int32_t* err,
                          cudaStream_t s) {
  const int n_tiles = perm_tiles(n_rows, TILE);
  dim3 grid(n_tiles, n_layers);
  hist_tiles_kernel<TILE><<<grid, kPermThreads, K * sizeof(int32_t), s>>>(ids, n_rows, K, n_tiles,
                                                                         counts, err);
  SIDA_LAUNCH_CHECK();
  // the scatter also publishes hist / off, so it runs even for zero rows;
  // programmatic dependent launch: its CTAs stage their ids while the
  // histogram grid drains and wait (griddepcontrol.wait) only before reading
  // the count matrix
  const size_t smem = (2ull * TILE + (size_t)(kPermWarps + 2) * K + 1) * sizeof(int32_t);
  static bool configured = false;
  if (!configured) {
    SIDA_CUDA(cudaFuncSetAttribute(scatter_kernel<TILE>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)((2ull * TILE + (kPermWarps + 2) * kMaxExperts + 1) *
                                         sizeof(int32_t))));
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kPermThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SIDA_CUDA(cudaLaunchKernelEx(&cfg, scatter_kernel<TILE>, ids, n_rows, K, n_tiles,
                               (const int32_t*)counts, alpha_rows, perm, inv, alpha_perm, hist,
                               off));
  count_launch();
  return SIDA_OK;
}

extern "C" int sida_permute_hist(const int32_t* ids, int n_layers, int n_rows, int num_experts,
                                 const float* alpha_rows, int32_t* hist, int32_t* off,
                                 int32_t* perm, int32_t* inv, float* alpha_perm, int32_t* err_flag,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  SIDA_REQUIRE(n_layers >= 1 && n_rows >= 0 && num_experts >= 1, SIDA_ERR_CONTRACT,
               "bad permute dims L=%d rows=%d K=%d", n_layers, n_rows, num_experts);
  SIDA_REQUIRE(num_experts <= kMaxExperts, SIDA_ERR_UNSUPPORTED, "K=%d > %d", num_experts,
               kMaxExperts);
  SIDA_REQUIRE(workspace_bytes >= sida_permute_workspace_bytes(n_layers, n_rows, num_experts),
               SIDA_ERR_CONTRACT, "permute workspace too small");
  SIDA_REQUIRE(!alpha_perm || alpha_rows, SIDA_ERR_CONTRACT, "alpha_perm needs alpha_rows");
  SIDA_REQUIRE(err_flag && hist && off && (n_rows == 0 || (ids && perm && inv)), SIDA_ERR_CONTRACT,
               "null pointer passed to sida_permute_hist");
  cudaStream_t s = as_stream(stream);
  const int tile = perm_tile(n_rows, n_layers);
  const size_t n = (size_t)n_layers * num_experts * perm_tiles(n_rows, tile);
  int32_t* counts = static_cast<int32_t*>(workspace);
  switch (tile) {
    case 1024: return permute_launch<1024>(ids, n_layers, n_rows, num_experts, alpha_rows, hist, off,
                                           perm, inv, alpha_perm, counts, err_flag, s);
    case 2048: return permute_launch<2048>(ids, n_layers, n_rows, num_experts, alpha_rows, hist, off,
                                           perm, inv, alpha_perm, counts, err_flag, s);
    case 4096: return permute_launch<4096>(ids, n_layers, n_rows, num_experts, alpha_rows, hist, off,
                                           perm, inv, alpha_perm, counts, err_flag, s);
    default: return permute_launch<8192>(ids, n_layers, n_rows, num_experts, alpha_rows, hist, off,
                                         perm, inv, alpha_perm, counts, err_flag, s);
  }
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
// alpha_rows (optional) replaces alpha_perm: the weight of (t, r) read in row
// order, for maps whose positions are not the table's permuted order (the
// chunk-major dispatch order of the expert-parallel NCCL path).
__global__ void __launch_bounds__(256)
unpermute_combine_kernel(const uint16_t* __restrict__ y_perm, const int32_t* __restrict__ inv,
                         const float* __restrict__ alpha_perm, const float* __restrict__ resid,
                         int n_tokens, int k, int d, float* __restrict__ out,
                         uint16_t* __restrict__ out_bf16,
                         const float* __restrict__ alpha_rows = nullptr) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_tokens; t += warps) {
    for (int c = lane * 4; c < d; c += 128) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int r = 0; r < k; ++r) {
        const int p = inv[(size_t)t * k + r];
        const float a = alpha_rows ? alpha_rows[(size_t)t * k + r] : alpha_perm[p];
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

extern "C" int sida_map_combine(const uint16_t* y, const int32_t* map, const float* alpha_rows,
                                const float* resid, int n_tokens, int k, int d, float* out,
                                uint16_t* out_bf16, void* stream) {
  SIDA_REQUIRE(d % 4 == 0 && k >= 1, SIDA_ERR_UNSUPPORTED, "combine needs d %% 4 == 0 (d=%d)", d);
  SIDA_REQUIRE(y && map && alpha_rows && resid && out, SIDA_ERR_CONTRACT,
               "null pointer passed to sida_map_combine");
  if (n_tokens == 0) return SIDA_OK;
  const int blocks = std::min(ceil_div(n_tokens, 8), kNumSMs * 16);
  unpermute_combine_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
      y, map, nullptr, resid, n_tokens, k, d, out, out_bf16, alpha_rows);
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
