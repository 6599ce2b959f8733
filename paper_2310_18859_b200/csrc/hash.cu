// SiDA hash function (expert-activation predictor), fp64, batched over every
// sequence of a batch. Replaces ref predictor.py:373-399 (build_hash_table,
// one Python call per sequence) over PredictorNet.forward
// (predictor.py:234-259). Runs in float64 like the reference so the top-k ids
// are bit-identical (SURVEY.md §7 "Bit-exact ids").
//
//   embed_xw1   emb = tok_emb[t] + pos_emb[pos] (fp64 of bf16 tables,
//               ref moe.py:218), comp = emb Wc + bc, xw1 = comp Wx1
//   lstm<H>     recurrence over each sequence (ref predictor.py:174-196):
//               gates = (xw_t + h Wh) + b, blocks i|f|g|o, Wh column per
//               thread in registers, S sequences per CTA
//   rows_gemm   xw2 = h1 Wx2, q/k/v = h2 W{q,k,v}
//   attn_heads  one warp per token: scores q.k (no 1/sqrt(H), :249),
//               per-row sparsemax by bitonic sort in smem (numkit.py:42-60),
//               ctx + h2 residual (:251-252), L heads, softmax over K,
//               top-k with ties to the lower index (numkit.py:87-93)
#include <algorithm>

#include "common.cuh"

namespace sida {
namespace hash {

constexpr int kMaxLen = 512;     // T_max supported by the smem sparsemax
constexpr int kMaxK = 1024;      // experts per layer
constexpr int kAttnWarps = 4;

struct Dims {
  int d, cd, H, L, K;
};

struct ParamPtrs {
  const double *cw, *cb, *wx1, *wh1, *b1, *wx2, *wh2, *b2, *wq, *wk, *wv, *hw, *hb;
};

__host__ __device__ inline ParamPtrs carve(const double* p, Dims dm) {
  ParamPtrs q;
  const int G = 4 * dm.H;
  q.cw = p; p += (size_t)dm.d * dm.cd;
  q.cb = p; p += dm.cd;
  q.wx1 = p; p += (size_t)dm.cd * G;
  q.wh1 = p; p += (size_t)dm.H * G;
  q.b1 = p; p += G;
  q.wx2 = p; p += (size_t)dm.H * G;
  q.wh2 = p; p += (size_t)dm.H * G;
  q.b2 = p; p += G;
  q.wq = p; p += (size_t)dm.H * dm.H;
  q.wk = p; p += (size_t)dm.H * dm.H;
  q.wv = p; p += (size_t)dm.H * dm.H;
  q.hw = p; p += (size_t)dm.L * dm.H * dm.K;
  q.hb = p;
  return q;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int seq_of(const int32_t* seq_off, int n_seq, int n) {
  int lo = 0, hi = n_seq - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (seq_off[mid] <= n) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ref numkit.py:104-110 (split branch for stability)
__device__ __forceinline__ double sigmoid_d(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}

// One warp per token: embedding (fp64 sum of bf16 tables), compress FC, and
// the layer-1 input projection xw1 = comp @ Wx1.
__global__ void __launch_bounds__(256)
embed_xw1_kernel(const uint16_t* __restrict__ tok_emb, const uint16_t* __restrict__ pos_emb,
                 const double* __restrict__ emb_f64, const int32_t* __restrict__ tokens, const int32_t* __restrict__ seq_off, int n_seq,
                 int n_tokens, Dims dm, ParamPtrs w, double* __restrict__ xw) {
  __shared__ double s_comp[8][64];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n = blockIdx.x * 8 + wib;
  if (n >= n_tokens) return;
  const int sq = seq_of(seq_off, n_seq, n);
  const int pos = n - seq_off[sq];
  const uint16_t* te = tok_emb ? tok_emb + (size_t)tokens[n] * dm.d : nullptr;
  const uint16_t* pe = tok_emb ? pos_emb + (size_t)pos * dm.d : nullptr;
  const double* ee = emb_f64 ? emb_f64 + (size_t)n * dm.d : nullptr;
  double part[64];
#pragma unroll
  for (int c = 0; c < 64; ++c) part[c] = 0.0;
  for (int j = lane; j < dm.d; j += 32) {
    const double e = ee ? ee[j] : (double)bf16_to_f32(te[j]) + (double)bf16_to_f32(pe[j]);
    const double* row = w.cw + (size_t)j * dm.cd;
#pragma unroll
    for (int c = 0; c < 64; ++c)
      if (c < dm.cd) part[c] = fma(e, row[c], part[c]);
  }
#pragma unroll
  for (int c = 0; c < 64; ++c) {
    if (c < dm.cd) {
      const double s = warp_sum(part[c]);
      if (lane == 0) s_comp[wib][c] = s + w.cb[c];
    }
  }
  __syncwarp();
  const int G = 4 * dm.H;
  for (int g = lane; g < G; g += 32) {
    double acc = 0.0;
    for (int c = 0; c < dm.cd; ++c) acc = fma(s_comp[wib][c], w.wx1[(size_t)c * G + g], acc);
    xw[(size_t)n * G + g] = acc;
  }
}

// LSTM recurrence. blockDim = 4H; thread g owns gate column g of Wh (in
// registers); S sequences per CTA share the weights.
template <int MAXH, int S>
__global__ void __launch_bounds__(4 * MAXH)
lstm_kernel(const double* __restrict__ xw, const double* __restrict__ wh, const double* __restrict__ b,
            const int32_t* __restrict__ seq_off, int n_seq, int H, double* __restrict__ h_out) {
  __shared__ double s_h[S][MAXH];
  __shared__ double s_gate[S][4 * MAXH];
  const int G = 4 * H;
  const int g = threadIdx.x;
  const int seq0 = blockIdx.x * S;
  double wcol[MAXH];
#pragma unroll
  for (int i = 0; i < MAXH; ++i) wcol[i] = (g < G && i < H) ? wh[(size_t)i * G + g] : 0.0;
  const double bg = g < G ? b[g] : 0.0;
  int len[S], base[S];
  int tmax = 0;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int sq = seq0 + s;
    base[s] = sq < n_seq ? seq_off[sq] : 0;
    len[s] = sq < n_seq ? seq_off[sq + 1] - seq_off[sq] : 0;
    tmax = max(tmax, len[s]);
  }
  // cell-update role: thread -> (sequence us, unit uj)
  const int us = g / MAXH, uj = g % MAXH;
  double c_state = 0.0;
  for (int i = threadIdx.x; i < S * MAXH; i += blockDim.x) (&s_h[0][0])[i] = 0.0;
  __syncthreads();
  for (int t = 0; t < tmax; ++t) {
    if (g < G) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (t < len[s]) {
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < MAXH; ++i)
            if (i < H) acc = fma(s_h[s][i], wcol[i], acc);
          s_gate[s][g] = (xw[(size_t)(base[s] + t) * G + g] + acc) + bg;
        }
      }
    }
    __syncthreads();
    if (us < S && uj < H && t < len[us]) {
      const double* gt = s_gate[us];
      const double ig = sigmoid_d(gt[uj]);
      const double fg = sigmoid_d(gt[H + uj]);
      const double gg = tanh(gt[2 * H + uj]);
      const double og = sigmoid_d(gt[3 * H + uj]);
      c_state = fg * c_state + ig * gg;
      const double hv = og * tanh(c_state);
      s_h[us][uj] = hv;
      h_out[(size_t)(base[us] + t) * H + uj] = hv;
    }
    __syncthreads();
  }
}

// C (N x M) = A (N x Kd) @ B (Kd x M), fp64; B staged in smem.
__global__ void __launch_bounds__(256)
rows_gemm_kernel(const double* __restrict__ A, int n_rows, int Kd, const double* __restrict__ B,
                 int M, double* __restrict__ C) {
  extern __shared__ double s_b[];
  for (int i = threadIdx.x; i < Kd * M; i += blockDim.x) s_b[i] = B[i];
  __syncthreads();
  const int rows_per_block = 16;
  const int r0 = blockIdx.x * rows_per_block;
  for (int i = threadIdx.x; i < rows_per_block * M; i += blockDim.x) {
    const int r = r0 + i / M, m = i % M;
    if (r >= n_rows) break;
    const double* a = A + (size_t)r * Kd;
    double acc = 0.0;
    for (int k = 0; k < Kd; ++k) acc = fma(a[k], s_b[k * M + m], acc);
    C[(size_t)r * M + m] = acc;
  }
}

// In-smem bitonic sort, descending, of n (power of two) doubles by one warp.
__device__ void warp_bitonic_desc(double* v, int n) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < n / 2; i += 32) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = ((lo & size) == 0);
        const double a = v[lo], b = v[hi];
        if (desc ? (a < b) : (a > b)) {
          v[lo] = b;
          v[hi] = a;
        }
      }
      __syncwarp();
    }
  }
}

// One warp per token: scores, sparsemax, ctx, residual, L heads, softmax,
// top-k. Smem per warp: scores[kMaxLen], sorted[kMaxLen], resid[64], z[kMaxK].
__global__ void __launch_bounds__(32 * kAttnWarps)
attn_heads_kernel(const double* __restrict__ q, const double* __restrict__ k,
                  const double* __restrict__ v, const double* __restrict__ h2,
                  const int32_t* __restrict__ seq_off, int n_seq, int n_tokens, Dims dm,
                  const double* __restrict__ hw, const double* __restrict__ hb, int topk,
                  int32_t* __restrict__ ids, double* __restrict__ alpha,
                  float* __restrict__ alpha_f32) {
  extern __shared__ double smem_d[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* s_sc = smem_d + (size_t)wib * (2 * kMaxLen + 64 + dm.K);
  double* s_srt = s_sc + kMaxLen;
  double* s_res = s_srt + kMaxLen;
  double* s_z = s_res + 64;
  const int H = dm.H;
  for (int n = blockIdx.x * kAttnWarps + wib; n < n_tokens; n += gridDim.x * kAttnWarps) {
    const int sq = seq_of(seq_off, n_seq, n);
    const int base = seq_off[sq], T = seq_off[sq + 1] - base;
    // q_n -> smem, then each lane owns score columns j = lane, lane+32, ...
    if (lane < H) s_res[lane] = q[(size_t)n * H + lane];
    if (lane + 32 < H) s_res[lane + 32] = q[(size_t)n * H + lane + 32];
    __syncwarp();
    int P = 1;
    while (P < T) P <<= 1;
    for (int j = lane; j < P; j += 32) {
      if (j < T) {
        const double* kr = k + (size_t)(base + j) * H;
        double sc = 0.0;
        for (int i = 0; i < H; ++i) sc = fma(s_res[i], kr[i], sc);
        s_sc[j] = sc;
        s_srt[j] = sc;
      } else {
        s_srt[j] = -INFINITY;
      }
    }
    __syncwarp();
    warp_bitonic_desc(s_srt, P);
    // running sum S_k of the sorted row (stored in place), support count
    // k_z = #{k : 1 + k z_(k) > S_k}, tau = (S_{k_z} - 1) / k_z (ref numkit.py:52-59)
    double carry = 0.0;
    int kz = 0;
    for (int c0 = 0; c0 < T; c0 += 32) {
      const int idx = c0 + lane;
      const double z = idx < T ? s_srt[idx] : 0.0;
      double incl = z;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const double S = carry + incl;
      const bool sup = idx < T && (1.0 + (double)(idx + 1) * z > S);
      kz += __popc(__ballot_sync(0xffffffffu, sup));
      if (idx < T) s_srt[idx] = S;
      carry = __shfl_sync(0xffffffffu, S, 31);
    }
    __syncwarp();
    const double tau = (s_srt[kz - 1] - 1.0) / (double)kz;
    // ctx = sum_j w_j v_j over the support; resid = ctx + h2_n
    double c0v = 0.0, c1v = 0.0;
    for (int j = 0; j < T; ++j) {
      const double wj = s_sc[j] - tau;
      if (wj > 0.0) {
        const double* vr = v + (size_t)(base + j) * H;
        if (lane < H) c0v = fma(wj, vr[lane], c0v);
        if (lane + 32 < H) c1v = fma(wj, vr[lane + 32], c1v);
      }
    }
    __syncwarp();  // every lane is done reading q from s_res
    if (lane < H) s_res[lane] = c0v + h2[(size_t)n * H + lane];
    if (lane + 32 < H) s_res[lane + 32] = c1v + h2[(size_t)n * H + lane + 32];
    __syncwarp();
    for (int l = 0; l < dm.L; ++l) {
      const double* W = hw + (size_t)l * H * dm.K;
      double zmax = -INFINITY;
      for (int e = lane; e < dm.K; e += 32) {
        double acc = 0.0;
        for (int i = 0; i < H; ++i) acc = fma(s_res[i], W[(size_t)i * dm.K + e], acc);
        const double z = acc + hb[(size_t)l * dm.K + e];
        s_z[e] = z;
        zmax = fmax(zmax, z);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
      double ssum = 0.0;
      for (int e = lane; e < dm.K; e += 32) {
        const double ex = exp(s_z[e] - zmax);
        s_z[e] = ex;
        ssum += ex;
      }
      ssum = warp_sum(ssum);
      __syncwarp();
      for (int e = lane; e < dm.K; e += 32) s_z[e] = s_z[e] / ssum;
      __syncwarp();
      // top-k on probabilities, descending, ties to the lower index
      for (int r = 0; r < topk; ++r) {
        double best = -1.0;
        int bi = 0x7fffffff;
        for (int e = lane; e < dm.K; e += 32) {
          const double pz = s_z[e];
          if (pz > best) { best = pz; bi = e; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) {
          const size_t at = ((size_t)l * n_tokens + n) * topk + r;
          ids[at] = bi;
          alpha[at] = best;
          if (alpha_f32) alpha_f32[at] = (float)best;
          s_z[bi] = -2.0;  // removed from later ranks
        }
        __syncwarp();
      }
    }
    __syncwarp();
  }
}

}  // namespace hash
}  // namespace sida

using namespace sida;
using namespace sida::hash;

static size_t ws_align(size_t b) { return align_up(b, 256); }

extern "C" size_t sida_hash_param_count(int d, int cd, int H, int L, int K) {
  const size_t G = 4ull * H;
  return (size_t)d * cd + cd + (size_t)cd * G + (size_t)H * G + G + 2ull * H * G + G +
         3ull * H * H + (size_t)L * H * K + (size_t)L * K;
}

extern "C" size_t sida_hash_workspace_bytes(int n_tokens, int n_seq, int max_len, int d, int cd,
                                            int H, int L, int K) {
  (void)n_seq; (void)max_len; (void)d; (void)cd; (void)L; (void)K;
  const size_t n = (size_t)n_tokens;
  return ws_align(n * 4 * H * 8) + 5 * ws_align(n * H * 8);
}

template <int MAXH>
static int launch_lstm(const double* xw, const double* wh, const double* b, const int32_t* seq_off,
                       int n_seq, int H, double* h_out, cudaStream_t s) {
  int S = 1;
  if (n_seq >= 4 * kNumSMs) S = 4;
  else if (n_seq >= 2 * kNumSMs) S = 2;
  if (S == 4)
    lstm_kernel<MAXH, 4><<<ceil_div(n_seq, 4), 4 * MAXH, 0, s>>>(xw, wh, b, seq_off, n_seq, H, h_out);
  else if (S == 2)
    lstm_kernel<MAXH, 2><<<ceil_div(n_seq, 2), 4 * MAXH, 0, s>>>(xw, wh, b, seq_off, n_seq, H, h_out);
  else
    lstm_kernel<MAXH, 1><<<n_seq, 4 * MAXH, 0, s>>>(xw, wh, b, seq_off, n_seq, H, h_out);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

static int lstm_dispatch(const double* xw, const double* wh, const double* b,
                         const int32_t* seq_off, int n_seq, int H, double* h_out, cudaStream_t s) {
  if (H <= 16) return launch_lstm<16>(xw, wh, b, seq_off, n_seq, H, h_out, s);
  if (H <= 32) return launch_lstm<32>(xw, wh, b, seq_off, n_seq, H, h_out, s);
  if (H <= 48) return launch_lstm<48>(xw, wh, b, seq_off, n_seq, H, h_out, s);
  return launch_lstm<64>(xw, wh, b, seq_off, n_seq, H, h_out, s);
}

static int rows_gemm(const double* A, int n, int Kd, const double* B, int M, double* C,
                     cudaStream_t s) {
  const size_t smem = (size_t)Kd * M * sizeof(double);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    SIDA_CUDA(cudaFuncSetAttribute(rows_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    configured = smem;
  }
  rows_gemm_kernel<<<ceil_div(n, 16), 256, smem, s>>>(A, n, Kd, B, M, C);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_hash_forward(const double* params, const uint16_t* tok_emb,
                                 const uint16_t* pos_emb, const double* emb_f64,
                                 const int32_t* tokens,
                                 const int32_t* seq_off, int n_seq, int n_tokens, int max_len,
                                 int d, int cd, int H, int L, int K, int topk, int32_t* ids,
                                 double* alpha, float* alpha_f32, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  SIDA_REQUIRE(topk >= 1 && topk <= K, SIDA_ERR_CONTRACT, "eval_top_k=%d out of range for K=%d",
               topk, K);
  SIDA_REQUIRE(n_seq >= 1 && n_tokens >= n_seq, SIDA_ERR_CONTRACT, "empty batch or sequence");
  SIDA_REQUIRE(H >= 1 && H <= 64 && cd >= 1 && cd <= 64, SIDA_ERR_UNSUPPORTED,
               "predictor dims cd=%d H=%d outside the kernel contract (<= 64)", cd, H);
  SIDA_REQUIRE(max_len <= kMaxLen, SIDA_ERR_UNSUPPORTED, "sequence length %d > %d", max_len,
               kMaxLen);
  SIDA_REQUIRE(K <= kMaxK, SIDA_ERR_UNSUPPORTED, "K=%d > %d", K, kMaxK);
  SIDA_REQUIRE(workspace_bytes >= sida_hash_workspace_bytes(n_tokens, n_seq, max_len, d, cd, H, L, K),
               SIDA_ERR_CONTRACT, "hash workspace too small");
  cudaStream_t s = as_stream(stream);
  Dims dm{d, cd, H, L, K};
  ParamPtrs w = carve(params, dm);
  const size_t n = (size_t)n_tokens;
  char* ws = static_cast<char*>(workspace);
  double* xw = reinterpret_cast<double*>(ws);
  ws += ws_align(n * 4 * H * 8);
  double* h1 = reinterpret_cast<double*>(ws); ws += ws_align(n * H * 8);
  double* h2 = reinterpret_cast<double*>(ws); ws += ws_align(n * H * 8);
  double* qb = reinterpret_cast<double*>(ws); ws += ws_align(n * H * 8);
  double* kb = reinterpret_cast<double*>(ws); ws += ws_align(n * H * 8);
  double* vb = reinterpret_cast<double*>(ws);

  SIDA_REQUIRE(emb_f64 || (tok_emb && pos_emb && tokens), SIDA_ERR_CONTRACT,
               "hash needs either embeddings or (tables, tokens)");
  embed_xw1_kernel<<<ceil_div(n_tokens, 8), 256, 0, s>>>(tok_emb, pos_emb, emb_f64, tokens, seq_off,
                                                         n_seq, n_tokens, dm, w, xw);
  SIDA_LAUNCH_CHECK();
  int st = lstm_dispatch(xw, w.wh1, w.b1, seq_off, n_seq, H, h1, s);
  if (st) return st;
  if ((st = rows_gemm(h1, n_tokens, H, w.wx2, 4 * H, xw, s))) return st;
  if ((st = lstm_dispatch(xw, w.wh2, w.b2, seq_off, n_seq, H, h2, s))) return st;
  if ((st = rows_gemm(h2, n_tokens, H, w.wq, H, qb, s))) return st;
  if ((st = rows_gemm(h2, n_tokens, H, w.wk, H, kb, s))) return st;
  if ((st = rows_gemm(h2, n_tokens, H, w.wv, H, vb, s))) return st;

  const size_t smem = (size_t)kAttnWarps * (2 * kMaxLen + 64 + K) * sizeof(double);
  static size_t configured = 0;
  if (smem > configured) {
    SIDA_CUDA(cudaFuncSetAttribute(attn_heads_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    configured = smem;
  }
  const int blocks = std::min(ceil_div(n_tokens, kAttnWarps), kNumSMs * 8);
  attn_heads_kernel<<<blocks, 32 * kAttnWarps, smem, s>>>(qb, kb, vb, h2, seq_off, n_seq, n_tokens,
                                                          dm, w.hw, w.hb, topk, ids, alpha,
                                                          alpha_f32);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}
