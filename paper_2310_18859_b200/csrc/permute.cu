// Token permute + histogram, every MoE layer of a
// batch in one launch chain, plus the bf16 row gather.
//
// The reference never permutes: moe_apply gathers w1[ids] per token
// (ref moe.py:253-256). The GPU path groups the (token, rank) rows of each
// layer by expert with a stable counting sort whose output is bit-identical
// to np.argsort(ids[l].reshape(-1), kind="stable") (oracle/permute.py).
// Rows are cut into tiles of TILE rows (1024 or 2048); three launches, the
// last two programmatically dependent on their predecessor:
//
//   rank_tiles  one CTA of 256 threads per (layer, tile): the tile's ids
//               staged in shared memory by 128-bit loads; each warp walks its
//               contiguous rows in order, the in-warp stable rank from the
//               mask of lanes with the same expert (one ballot per id bit)
//               + popc and per-warp running counts per expert; a per-expert prefix over the warps turns them into
//               the row's rank among the tile's rows of its expert. Writes
//               the tile's per-expert counts and one code per row
//               (expert | rank << 10), both coalesced.
//   tile_base   one CTA per (32 experts, layer), threads = (tile chunk,
//               expert): the exclusive scan of the counts over tiles (each
//               (tile, expert) run's offset inside its expert) -> base, hist.
//   place_tiles (below) also scans hist over experts with warp-shuffle
//               prefix sums for the expert offsets (tile 0 publishes off).
//   place_tiles one CTA per (layer, tile): position of row r = off[e] +
//               base[tile][e] + rank; inv written row-ordered (coalesced),
//               the tile's rows staged in shared memory in sorted order so
//               that perm / alpha_perm are written as contiguous runs per
//               (tile, expert).
//
// Every row's expert is matched once (the rank pass), and no CTA re-reads
// the count matrix column of its layer.
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
constexpr int kRankShift = 10;  // code = expert | rank_in_tile << 10 (K <= 1024, TILE <= 2^21)

// Tile rows for (rows, layers): 2048, or 1024 when that is needed for ~2 CTAs per SM.
static inline int perm_tile(int n_rows, int n_layers) {
  const long long work = (long long)n_rows * std::max(n_layers, 1);
  return work >= 2048ll * 2 * kNumSMs ? 2048 : 1024;
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

// Lanes of the warp holding the same key as this lane (keys in [0, 2^nbits)
// or -1): one ballot per key bit plus one for validity. The same mask as
// __match_any_sync, without its serialised MIO-pipe cost (ncu: MATCH bound
// the rank pass at ~90 cycles per warp instruction per SM).
__device__ __forceinline__ unsigned lanes_with_key(int e, int nbits) {
  const bool valid = e >= 0;
  const unsigned vb = __ballot_sync(0xffffffffu, valid);
  unsigned m = valid ? vb : ~vb;
  for (int b = 0; b < nbits; ++b) {
    const bool bit = (e >> b) & 1;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bal : ~bal;
  }
  return m;
}

template <int TILE>
__global__ void __launch_bounds__(kPermThreads)
rank_tiles_kernel(const int32_t* __restrict__ ids, int n_rows, int K, int n_tiles,
                  int32_t* __restrict__ counts, int32_t* __restrict__ codes,
                  int32_t* __restrict__ err) {
  constexpr int R = TILE / kPermWarps;  // contiguous rows per warp
  constexpr int NR = R / 32;            // rounds per warp
  extern __shared__ int32_t smem[];
  int32_t* s_ids = smem;          // [TILE]
  int32_t* s_cnt = s_ids + TILE;  // [warps][K] counts -> warp prefix
  const int layer = blockIdx.y, tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = tile * TILE, r1 = min(n_rows, r0 + TILE), n = r1 - r0;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int i = threadIdx.x; i < kPermWarps * K; i += blockDim.x) s_cnt[i] = 0;
  stage_ids(ids + (size_t)layer * n_rows, r0, r1, s_ids);
  __syncthreads();

  // in-order stable ranks, per warp over its R rows
  const unsigned lt = (1u << lane) - 1u;
  int32_t* my_cnt = s_cnt + warp * K;
  int nbits = 0;
  while ((1 << nbits) < K) ++nbits;
  int loc[NR];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int i = warp * R + j * 32 + lane;
    int e = i < n ? s_ids[i] : -1;
    if (i < n && (e < 0 || e >= K)) { bad = true; e = -1; }
    const unsigned peers = lanes_with_key(e, nbits);
    int base = 0;
    if (e >= 0) base = my_cnt[e];
    __syncwarp();
    if (e >= 0 && (peers & lt) == 0) my_cnt[e] = base + __popc(peers);
    __syncwarp();
    loc[j] = base + __popc(peers & lt);
  }
  if (bad) atomicExch(err, 1);
  __syncthreads();
  // warp prefix per expert (in place); the tile's per-expert totals
  int32_t* c = counts + ((size_t)layer * n_tiles + tile) * K;
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < kPermWarps; ++w) {
      const int v = s_cnt[w * K + e];
      s_cnt[w * K + e] = run;
      run += v;
    }
    c[e] = run;
  }
  __syncthreads();
  int32_t* lcode = codes + (size_t)layer * n_rows + r0;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int i = warp * R + j * 32 + lane;
    if (i < n) {
      const int e = s_ids[i];
      lcode[i] = (e >= 0 && e < K) ? (e | ((s_cnt[warp * K + e] + loc[j]) << kRankShift)) : -1;
    }
  }
}

// CTA (32 experts, layer), 1024 threads: thread (q, e) owns expert e's counts
// over the q-th of 32 contiguous tile chunks: chunk sums, a prefix over the
// chunks in shared memory, then base[l][t][e] = sum of counts[l][t'][e] over
// t' < t, and hist[l][e] = the expert's total. Warp = 32 consecutive experts of
// one chunk, so every counts / base access is a coalesced 128 B row segment.
// (The expert offsets -- a scan of hist over experts -- are taken by
// place_tiles, which needs them per CTA anyway.)
__global__ void __launch_bounds__(1024)
tile_base_kernel(const int32_t* __restrict__ counts, int K, int n_tiles, int32_t* __restrict__ base,
                 int32_t* __restrict__ hist) {
  __shared__ int s_part[32][33];
  const int layer = blockIdx.y;
  const int el = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + el;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // rank_tiles' counts are complete
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int32_t* cl = counts + (size_t)layer * n_tiles * K;
  int32_t* bl = base + (size_t)layer * n_tiles * K;
  const int t0 = q * n_tiles / 32, t1 = (q + 1) * n_tiles / 32;
  const bool mine = e < K;
  int sum = 0;
  if (mine)
    for (int t = t0; t < t1; ++t) sum += cl[(size_t)t * K + e];
  s_part[q][el] = sum;
  __syncthreads();
  int run = 0, tot = 0;
#pragma unroll 8
  for (int r = 0; r < 32; ++r) {
    const int v = s_part[r][el];
    run += r < q ? v : 0;
    tot += v;
  }
  if (mine) {
    for (int t = t0; t < t1; ++t) {
      const int v = cl[(size_t)t * K + e];
      bl[(size_t)t * K + e] = run;
      run += v;
    }
    if (q == 0) hist[(size_t)layer * K + e] = tot;
  }
}

template <int TILE>
__global__ void __launch_bounds__(kPermThreads)
place_tiles_kernel(const int32_t* __restrict__ codes, int n_rows, int K, int n_tiles,
                   const int32_t* __restrict__ counts, const int32_t* __restrict__ base,
                   const int32_t* __restrict__ hist, int32_t* __restrict__ off,
                   const float* __restrict__ alpha_rows, int32_t* __restrict__ perm,
                   int32_t* __restrict__ inv, float* __restrict__ alpha_perm) {
  extern __shared__ int32_t smem[];
  int32_t* s_code = smem;              // [TILE]
  int32_t* s_ord = s_code + TILE;      // [TILE] tile row of sorted position q
  int32_t* s_pos0 = s_ord + TILE;      // [K] first output position of (tile, e)
  int32_t* s_texc = s_pos0 + K;        // [K + 1] tile-local exclusive prefix
  const int layer = blockIdx.y, tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = tile * TILE, r1 = min(n_rows, r0 + TILE), n = r1 - r0;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // codes, counts, base, hist complete
  stage_ids(codes + (size_t)layer * n_rows, r0, r1, s_code);
  const size_t ct = ((size_t)layer * n_tiles + tile) * K;
  for (int e = threadIdx.x; e < K; e += blockDim.x) {
    s_texc[e] = counts[ct + e];
    s_pos0[e] = hist[(size_t)layer * K + e];  // -> expert offsets below
  }
  __syncthreads();
  if (warp == 1) {  // expert offsets: exclusive scan of the layer's histogram
    int carry = 0;
    for (int b = 0; b < K; b += 32) {
      const int e = b + lane;
      const int v = e < K ? s_pos0[e] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (e < K) {
        s_pos0[e] = carry + incl - v;
        if (tile == 0) off[(size_t)layer * (K + 1) + e] = carry + incl - v;
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tile == 0 && lane == 0) off[(size_t)layer * (K + 1) + K] = carry;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < K; e += blockDim.x) s_pos0[e] += base[ct + e];
  if (warp == 0) {  // exclusive scan of the tile's counts over experts
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
  int32_t* linv = inv + (size_t)layer * n_rows + r0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int code = s_code[i];
    if (code >= 0) {
      const int e = code & (kMaxExperts - 1), w = code >> kRankShift;
      linv[i] = s_pos0[e] + w;
      s_ord[s_texc[e] + w] = i;
    } else {
      linv[i] = -1;
    }
  }
  __syncthreads();
  const int n_valid = s_texc[K];
  int32_t* lperm = perm + (size_t)layer * n_rows;
  const float* la = alpha_rows ? alpha_rows + (size_t)layer * n_rows + r0 : nullptr;
  float* lap = alpha_perm ? alpha_perm + (size_t)layer * n_rows : nullptr;
  for (int q = threadIdx.x; q < n_valid; q += blockDim.x) {
    const int i = s_ord[q];
    const int e = s_code[i] & (kMaxExperts - 1);
    const int pos = s_pos0[e] + (q - s_texc[e]);
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
  const size_t n = (size_t)n_layers * num_experts * perm_tiles(n_rows, tile);
  return 2 * align_up(n * sizeof(int32_t), 256) +
         align_up((size_t)n_layers * std::max(n_rows, 1) * sizeof(int32_t), 256);
}

template <typename Kern, typename... Args>
static int launch_pdl(Kern kern, dim3 grid, int threads, size_t smem, cudaStream_t s,
                      Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SIDA_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
  count_launch();
  return SIDA_OK;
}

template <int TILE>
static int permute_launch(const int32_t* ids, int n_layers, int n_rows, int K, const float* alpha_rows,
                          int32_t* hist, int32_t* off, int32_t* perm, int32_t* inv,
                          float* alpha_perm, void* workspace, int32_t* err, cudaStream_t s) {
  const int n_tiles = perm_tiles(n_rows, TILE);
  const size_t n = (size_t)n_layers * K * n_tiles;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  int32_t* counts = reinterpret_cast<int32_t*>(ws);
  int32_t* base = reinterpret_cast<int32_t*>(ws + align_up(n * sizeof(int32_t), 256));
  int32_t* codes = reinterpret_cast<int32_t*>(ws + 2 * align_up(n * sizeof(int32_t), 256));
  const dim3 grid(n_tiles, n_layers);
  const size_t smem1 = ((size_t)TILE + (size_t)kPermWarps * K) * sizeof(int32_t);
  const size_t smem3 = (2ull * TILE + 2ull * K + 1) * sizeof(int32_t);
  static bool configured = false;
  if (!configured) {
    SIDA_CUDA(cudaFuncSetAttribute(rank_tiles_kernel<TILE>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(((size_t)TILE + (size_t)kPermWarps * kMaxExperts) *
                                         sizeof(int32_t))));
    configured = true;
  }
  if (n_rows > 0) {
    rank_tiles_kernel<TILE><<<grid, kPermThreads, smem1, s>>>(ids, n_rows, K, n_tiles, counts, codes,
                                                              err);
    SIDA_LAUNCH_CHECK();
  } else {
    SIDA_CUDA(cudaMemsetAsync(counts, 0, n * sizeof(int32_t), s));
  }
  // tile_base publishes hist / off, so it runs even for zero rows
  int st = launch_pdl(tile_base_kernel, dim3(ceil_div(K, 32), n_layers), 1024, 0, s,
                      (const int32_t*)counts, K, n_tiles, base, hist);
  if (st) return st;
  if (n_rows == 0) {  // no tiles to place: publish the (all-zero) offsets
    SIDA_CUDA(cudaMemsetAsync(off, 0, (size_t)n_layers * (K + 1) * sizeof(int32_t), s));
    return SIDA_OK;
  }
  return launch_pdl(place_tiles_kernel<TILE>, grid, kPermThreads, smem3, s, (const int32_t*)codes,
                    n_rows, K, n_tiles, (const int32_t*)counts, (const int32_t*)base,
                    (const int32_t*)hist, off, alpha_rows, perm, inv, alpha_perm);
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
  SIDA_REQUIRE(workspace && ((uintptr_t)workspace & 255) == 0, SIDA_ERR_CONTRACT,
               "permute workspace must be 256-byte aligned");
  cudaStream_t s = as_stream(stream);
  if (perm_tile(n_rows, n_layers) == 2048)
    return permute_launch<2048>(ids, n_layers, n_rows, num_experts, alpha_rows, hist, off, perm,
                                inv, alpha_perm, workspace, err_flag, s);
  return permute_launch<1024>(ids, n_layers, n_rows, num_experts, alpha_rows, hist, off, perm, inv,
                              alpha_perm, workspace, err_flag, s);
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
