// SiDA hash function (expert-activation predictor), fp64, batched over every
// sequence of a batch. Replaces ref predictor.py:373-399 (build_hash_table,
// one Python call per sequence) over PredictorNet.forward
// (predictor.py:234-259). Runs in float64 like the reference so the top-k ids
// are bit-identical (SURVEY.md §7 "Bit-exact ids").
//
// Per-vocabulary folding (sida_hash_prepare, once per model + predictor):
// the layer-1 LSTM input x_t Wx1 = (emb_t Wc + bc) Wx1 is linear in the
// embedding emb_t = tok_emb[t] + pos_emb[p] (ref moe.py:218), so it splits
// into  TX[t] + PX[p] + bc Wx1  with TX = (tok_emb Wc) Wx1 (vocab x 4H) and
// PX = (pos_emb Wc) Wx1 (max_len x 4H), both computed once in fp64. Per batch
// the compress FC and the input projection become two table rows.
//
//   lstm<H,S>   recurrence over each sequence (ref predictor.py:174-196):
//               gates = (x_t Wx + h Wh) + b, blocks i|f|g|o, the Wh column of
//               each gate in registers, four independent FMA chains
//   rows_gemm   xw2 = h1 Wx2 and qkv = h2 [Wq|Wk|Wv], smem-tiled, 4x6
//               register blocking
//   attn_heads  CTA per (sequence, 32-query block): K staged in smem
//               (transposed), one warp per query row: scores q.k (no
//               1/sqrt(H), :249), sparsemax by an smem bitonic sort
//               (numkit.py:42-60), ctx over the support + h2 residual
//               (:251-252), all L heads, softmax over K and top-k with ties to
//               the lower index (numkit.py:87-93)
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace sida {
namespace hash {

constexpr int kMaxLen = 512;     // T_max supported by the smem sparsemax
constexpr int kMaxK = 1024;      // experts per layer
constexpr int kAttnWarps = 8;
constexpr int kRowsPerBlk = 64;  // query rows per attention CTA (K/V staged once)

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

// One warp per row: out[row] = ((src[row] (+ pos_src[pos]) ) Wc (+ bc)) Wx1.
// Modes: table rows (bf16 source, no bias: vocabulary / position folding) or
// caller embeddings (fp64 source, with bias: the embed_fn path).
__global__ void __launch_bounds__(256)
project_rows_kernel(const uint16_t* __restrict__ tab_bf16, const double* __restrict__ emb_f64,
                    int n_rows, Dims dm, const double* __restrict__ cw,
                    const double* __restrict__ cb, const double* __restrict__ wx1,
                    double* __restrict__ out) {
  __shared__ double s_comp[8][64];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n = blockIdx.x * 8 + wib;
  if (n >= n_rows) return;
  double part[64];
#pragma unroll
  for (int c = 0; c < 64; ++c) part[c] = 0.0;
  for (int j = lane; j < dm.d; j += 32) {
    const double e = tab_bf16 ? (double)bf16_to_f32(tab_bf16[(size_t)n * dm.d + j])
                              : emb_f64[(size_t)n * dm.d + j];
    const double* row = cw + (size_t)j * dm.cd;
#pragma unroll
    for (int c = 0; c < 64; ++c)
      if (c < dm.cd) part[c] = fma(e, row[c], part[c]);
  }
#pragma unroll
  for (int c = 0; c < 64; ++c) {
    if (c < dm.cd) {
      const double s = warp_sum(part[c]);
      if (lane == 0) s_comp[wib][c] = cb ? s + cb[c] : s;
    }
  }
  __syncwarp();
  const int G = 4 * dm.H;
  for (int g = lane; g < G; g += 32) {
    double acc = 0.0;
    for (int c = 0; c < dm.cd; ++c) acc = fma(s_comp[wib][c], wx1[(size_t)c * G + g], acc);
    out[(size_t)n * G + g] = acc;
  }
}

// cX[g] = sum_c bc[c] Wx1[c][g] (the bias part of the folded input projection)
__global__ void bias_project_kernel(const double* __restrict__ cb, const double* __restrict__ wx1,
                                    int cd, int G, double* __restrict__ out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  double acc = 0.0;
  for (int c = 0; c < cd; ++c) acc = fma(cb[c], wx1[(size_t)c * G + g], acc);
  out[g] = acc;
}

// LSTM recurrence. blockDim = 4*MAXH; thread g owns gate column g of Wh (in
// registers); S sequences per CTA share the weights. Layer-1 input comes from
// the folded tables (FOLD) or a materialised x Wx (xw).
template <int MAXH, int S, bool FOLD>
__global__ void __launch_bounds__(4 * MAXH)
lstm_kernel(const double* __restrict__ xw, const double* __restrict__ tokx,
            const double* __restrict__ posx, const double* __restrict__ cx,
            const int32_t* __restrict__ tokens, const double* __restrict__ wh,
            const double* __restrict__ b, const int32_t* __restrict__ seq_off, int n_seq, int H,
            double* __restrict__ h_out) {
  __shared__ double s_h[S][MAXH];
  __shared__ double s_gate[S][4 * MAXH];
  const int G = 4 * H;
  const int g = threadIdx.x;
  const int seq0 = blockIdx.x * S;
  double wcol[MAXH];
#pragma unroll
  for (int i = 0; i < MAXH; ++i) wcol[i] = (g < G && i < H) ? wh[(size_t)i * G + g] : 0.0;
  const double bg = g < G ? b[g] : 0.0;
  const double cg = (FOLD && g < G) ? cx[g] : 0.0;
  int len[S], base[S];
  int tmax = 0;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int sq = seq0 + s;
    base[s] = sq < n_seq ? seq_off[sq] : 0;
    len[s] = sq < n_seq ? seq_off[sq + 1] - seq_off[sq] : 0;
    tmax = max(tmax, len[s]);
  }
  const int us = g / MAXH, uj = g % MAXH;  // cell-update role: (sequence, unit)
  double c_state = 0.0;
  for (int i = threadIdx.x; i < S * MAXH; i += blockDim.x) (&s_h[0][0])[i] = 0.0;
  __syncthreads();
  // x_t Wx does not depend on h, so it is fetched ahead of the recurrence:
  // the token id two steps ahead, its table row (and the position row) one
  // step ahead, and the parts are only added when the step consumes them --
  // the dependent id -> row load chain stays off the critical path.
  auto tok_at = [&](int s, int t) -> int {
    return (FOLD && g < G && t < len[s]) ? __ldg(tokens + base[s] + t) : 0;
  };
  auto load_parts = [&](int s, int t, int tok, double& pa, double& pb) {
    pa = pb = 0.0;
    if (g >= G || t >= len[s]) return;
    if (FOLD) {
      pa = __ldg(tokx + (size_t)tok * G + g);
      pb = __ldg(posx + (size_t)t * G + g);
    } else {
      pa = __ldg(xw + (size_t)(base[s] + t) * G + g);
    }
  };
  double xa[S], xb[S];
  int tok1[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    load_parts(s, 0, tok_at(s, 0), xa[s], xb[s]);
    tok1[s] = tok_at(s, 1);
  }
  for (int t = 0; t < tmax; ++t) {
    double xcur[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      xcur[s] = FOLD ? (xa[s] + xb[s]) + cg : xa[s];
      const int tok2 = tok_at(s, t + 2);
      load_parts(s, t + 1, tok1[s], xa[s], xb[s]);
      tok1[s] = tok2;
    }
    if (g < G) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (t < len[s]) {
          const double x = xcur[s];
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int i = 0; i < MAXH; i += 4) {
            if (i < H) a0 = fma(s_h[s][i], wcol[i], a0);
            if (i + 1 < H) a1 = fma(s_h[s][i + 1], wcol[i + 1], a1);
            if (i + 2 < H) a2 = fma(s_h[s][i + 2], wcol[i + 2], a2);
            if (i + 3 < H) a3 = fma(s_h[s][i + 3], wcol[i + 3], a3);
          }
          const double pre = (x + ((a0 + a1) + (a2 + a3))) + bg;
          // gate nonlinearity on the gate's own thread: i, f, o sigmoid; g tanh
          s_gate[s][g] = (g >= 2 * H && g < 3 * H) ? tanh(pre) : sigmoid_d(pre);
        }
      }
    }
    __syncthreads();
    if (us < S && uj < H && t < len[us]) {
      const double* gt = s_gate[us];
      const double ig = gt[uj], fg = gt[H + uj], gg = gt[2 * H + uj], og = gt[3 * H + uj];
      c_state = fg * c_state + ig * gg;
      const double hv = og * tanh(c_state);
      s_h[us][uj] = hv;
      h_out[(size_t)(base[us] + t) * H + uj] = hv;
    }
    __syncthreads();
  }
}

// Gate / cell nonlinearity without divergence: sigmoid (ref numkit.py:104-110,
// stable split) or tanh from one expm1 and one division,
//   m = expm1(-a|x|), a = 1 (sigmoid) or 2 (tanh):
//   sigmoid(x >= 0) = 1 / (2 + m), sigmoid(x < 0) = (1 + m) / (2 + m),
//   tanh(x) = sign(x) * (-m) / (2 + m)            (expm1 keeps tanh accurate near 0)
__device__ __forceinline__ double act_d(double x, bool is_tanh) {
  const double ax = fabs(x);
  const double m = expm1(is_tanh ? -2.0 * ax : -ax);
  const double num = is_tanh ? -m : (x >= 0.0 ? 1.0 : 1.0 + m);
  const double r = num / (2.0 + m);
  return (is_tanh && x < 0.0) ? -r : r;
}

// LSTM recurrence, one sequence per CTA, quad mapping: thread t owns gate
// q = t % 4 (i, f, g, o) of unit j = t / 4, i.e. column q*H + j of Wh (in
// registers) and Wx. The four gates of a unit sit in one lane quad, so the
// cell update c = f c + i g, h = o tanh(c) needs two shuffles and no shared
// memory; one barrier per step publishes h. (ref predictor.py:174-196)
template <int H, bool FOLD>
__global__ void __launch_bounds__(4 * H)
lstm_quad_kernel(const double* __restrict__ xw, const double* __restrict__ tokx,
                 const double* __restrict__ posx, const double* __restrict__ cx,
                 const int32_t* __restrict__ tokens, const double* __restrict__ wh,
                 const double* __restrict__ b, const int32_t* __restrict__ seq_off, int n_seq,
                 double* __restrict__ h_out, int t0, int t1, double* __restrict__ c_buf) {
  // steps [t0, t1) of every sequence: the recurrence is cut into short
  // launches (state c in c_buf, h from h_out) so its CTAs never hold SMs for
  // long -- the persistent compute-stream GEMMs then find their SMs free
  constexpr int G = 4 * H;
  __shared__ double s_h[2][H];
  const int t = threadIdx.x;
  const int j = t >> 2, q = t & 3;
  const int col = q * H + j;
  const bool is_tanh = q == 2;
  const int seq = blockIdx.x;
  const int base = seq_off[seq];
  const int len = seq_off[seq + 1] - base;
  if (t0 >= len) return;  // (uniform per CTA, before any barrier)
  const int tend = min(t1, len);
  double wcol[H];
#pragma unroll
  for (int i = 0; i < H; ++i) wcol[i] = wh[(size_t)i * G + col];
  const double bg = b[col];
  const double cg = FOLD ? cx[col] : 0.0;
  for (int i = t; i < H; i += blockDim.x)
    s_h[t0 & 1][i] = t0 > 0 ? h_out[(size_t)(base + t0 - 1) * H + i] : 0.0;
  double c_state = t0 > 0 ? c_buf[(size_t)seq * H + j] : 0.0;
  // x_t fetched ahead: token ids two steps, table rows one step (see lstm_kernel)
  auto tok_at = [&](int tt) -> int { return (FOLD && tt < len) ? __ldg(tokens + base + tt) : 0; };
  double xa = 0.0, xb = 0.0;
  auto load_parts = [&](int tt, int tok) {
    xa = xb = 0.0;
    if (tt >= len) return;
    if (FOLD) {
      xa = __ldg(tokx + (size_t)tok * G + col);
      xb = __ldg(posx + (size_t)tt * G + col);
    } else {
      xa = __ldg(xw + (size_t)(base + tt) * G + col);
    }
  };
  load_parts(t0, tok_at(t0));
  int tok1 = tok_at(t0 + 1);
  __syncthreads();
  for (int tt = t0; tt < tend; ++tt) {
    const double* hp = s_h[tt & 1];
    const double x = FOLD ? (xa + xb) + cg : xa;
    const int tok2 = tok_at(tt + 2);
    load_parts(tt + 1, tok1);
    tok1 = tok2;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int i = 0; i < H; i += 4) {
      a0 = fma(hp[i], wcol[i], a0);
      if (i + 1 < H) a1 = fma(hp[i + 1], wcol[i + 1], a1);
      if (i + 2 < H) a2 = fma(hp[i + 2], wcol[i + 2], a2);
      if (i + 3 < H) a3 = fma(hp[i + 3], wcol[i + 3], a3);
    }
    const double pre = (x + ((a0 + a1) + (a2 + a3))) + bg;
    const double gv = act_d(pre, is_tanh);
    // gather the unit's i, f, g, o inside the quad (every lane gets all four)
    const double gi = __shfl_sync(0xffffffffu, gv, 0, 4);
    const double gf = __shfl_sync(0xffffffffu, gv, 1, 4);
    const double gg = __shfl_sync(0xffffffffu, gv, 2, 4);
    const double go = __shfl_sync(0xffffffffu, gv, 3, 4);
    c_state = gf * c_state + gi * gg;
    const double hv = go * act_d(c_state, true);
    if (q == 0) {
      s_h[(tt + 1) & 1][j] = hv;
      h_out[(size_t)(base + tt) * H + j] = hv;
    }
    __syncthreads();
  }
  if (q == 0 && tend < len) c_buf[(size_t)seq * H + j] = c_state;
}

// C (N x M) = A (N x Kd) @ B (Kd x M), fp64. Block = 64 rows; A and B in smem;
// 256 threads as a 16 x 16 grid, each 4 rows x (M/16) columns.
constexpr int kRG_Rows = 64;
__global__ void __launch_bounds__(256)
rows_gemm_kernel(const double* __restrict__ A, int n_rows, int Kd, const double* __restrict__ B,
                 int M, double* __restrict__ C) {
  extern __shared__ double smem_d[];
  double* s_b = smem_d;                  // Kd x M
  double* s_a = smem_d + (size_t)Kd * M; // 64 x (Kd + 1)
  const int r0 = blockIdx.x * kRG_Rows;
  for (int i = threadIdx.x; i < Kd * M; i += blockDim.x) s_b[i] = B[i];
  for (int i = threadIdx.x; i < kRG_Rows * Kd; i += blockDim.x) {
    const int r = i / Kd, k = i % Kd;
    s_a[r * (Kd + 1) + k] = (r0 + r < n_rows) ? A[(size_t)(r0 + r) * Kd + k] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int ncol = (M + 15) / 16;  // <= 12
  double acc[4][12];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 12; ++j) acc[i][j] = 0.0;
  for (int k = 0; k < Kd; ++k) {
    double a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = s_a[(ty * 4 + i) * (Kd + 1) + k];
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      if (j < ncol && tx + 16 * j < M) {
        const double bv = s_b[k * M + tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][j] = fma(a[i], bv, acc[i][j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty * 4 + i;
    if (r >= n_rows) continue;
#pragma unroll
    for (int j = 0; j < 12; ++j)
      if (j < ncol && tx + 16 * j < M) C[(size_t)r * M + tx + 16 * j] = acc[i][j];
  }
}

// Top-k helper: (value desc, index asc) arg-max over a group of W lanes.
__device__ __forceinline__ void seg_argmax(double& best, int& bi, int W) {
  for (int o = W >> 1; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
}

struct AttnArgs {
  const double* qkv;   // (N, 3H): q | k | v
  const double* h2;    // (N, H)
  const int32_t* seq_off;
  const int32_t* blk_off;  // (n_seq+1) prefix of ceil(len/kRowsPerBlk)
  int n_seq, n_tokens;
  Dims dm;
  const double* hw;
  const double* hb;
  int topk;
  int32_t* ids;
  double* alpha;
  float* alpha_f32;
  unsigned long long* prof;  // optional per-warp phase cycles (SIDA_HASH_PROF)
  int ts;  // keys/values staged in smem per sequence (0: read them from L2)
};

constexpr int kMaxZ = kMaxLen / 32;  // score registers per lane
constexpr int kResPitch = 49;         // smem pitch (doubles) of a residual row: conflict-free

// Record the selected (id, probability) of rank r for (layer, token n).
__device__ __forceinline__ void emit(const AttnArgs& a, int l, int n, int r, int id, double p) {
  const size_t at = ((size_t)l * a.n_tokens + n) * a.topk + r;
  a.ids[at] = id;
  a.alpha[at] = p;
  if (a.alpha_f32) a.alpha_f32[at] = (float)p;
}

// Heads for small K: one thread per (row, layer); the K logits stay in
// registers; softmax over K (ref numkit.py:28-33) then top-k on the
// probabilities, descending, ties to the lower index (numkit.py:87-93).
template <int KB>
__device__ void heads_small(const AttnArgs& a, const double* s_res, int rows, int n0) {
  const int H = a.dm.H, K = a.dm.K, L = a.dm.L;
  for (int pr = threadIdx.x; pr < rows * L; pr += blockDim.x) {
    const int r = pr / L, l = pr % L;
    const double* res = s_res + r * kResPitch;
    const double* W = a.hw + (size_t)l * H * K;
    double z[KB];
#pragma unroll
    for (int e = 0; e < KB; ++e) z[e] = 0.0;
    for (int i = 0; i < H; ++i) {
      const double ri = res[i];
      const double* wr = W + (size_t)i * K;
#pragma unroll
      for (int e = 0; e < KB; ++e)
        if (e < K) z[e] = fma(ri, wr[e], z[e]);
    }
    double zmax = -INFINITY;
#pragma unroll
    for (int e = 0; e < KB; ++e)
      if (e < K) {
        z[e] += a.hb[(size_t)l * K + e];
        zmax = fmax(zmax, z[e]);
      }
    double ssum = 0.0;
#pragma unroll
    for (int e = 0; e < KB; ++e)
      if (e < K) {
        z[e] = exp(z[e] - zmax);
        ssum += z[e];
      }
#pragma unroll
    for (int e = 0; e < KB; ++e)
      if (e < K) z[e] = z[e] / ssum;
    for (int rk = 0; rk < a.topk; ++rk) {
      double best = -1.0;
      int bi = 0;
#pragma unroll
      for (int e = 0; e < KB; ++e)
        if (e < K && z[e] > best) { best = z[e]; bi = e; }
      emit(a, l, n0 + r, rk, bi, best);
#pragma unroll
      for (int e = 0; e < KB; ++e)
        if (e == bi) z[e] = -2.0;  // removed from later ranks
    }
  }
}

// Heads for large K: one warp per (row, layer), lanes over experts, MZ
// logits per lane in registers.
template <int MZ>
__device__ void heads_large(const AttnArgs& a, const double* s_res, int rows, int n0) {
  const int H = a.dm.H, K = a.dm.K, L = a.dm.L;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int pr = wib; pr < rows * L; pr += kAttnWarps) {
    const int r = pr / L, l = pr % L;
    const double* res = s_res + r * kResPitch;
    const double* W = a.hw + (size_t)l * H * K;
    double z[MZ];
#pragma unroll
    for (int m = 0; m < MZ; ++m) z[m] = 0.0;
    for (int i = 0; i < H; ++i) {
      const double ri = res[i];
      const double* wr = W + (size_t)i * K + lane;
#pragma unroll
      for (int m = 0; m < MZ; ++m)
        if (lane + 32 * m < K) z[m] = fma(ri, wr[32 * m], z[m]);
    }
    double zmax = -INFINITY;
#pragma unroll
    for (int m = 0; m < MZ; ++m)
      if (lane + 32 * m < K) {
        z[m] += a.hb[(size_t)l * K + lane + 32 * m];
        zmax = fmax(zmax, z[m]);
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
    double ssum = 0.0;
#pragma unroll
    for (int m = 0; m < MZ; ++m)
      if (lane + 32 * m < K) {
        z[m] = exp(z[m] - zmax);
        ssum += z[m];
      }
    ssum = warp_sum(ssum);
#pragma unroll
    for (int m = 0; m < MZ; ++m) z[m] = lane + 32 * m < K ? z[m] / ssum : -2.0;
    for (int rk = 0; rk < a.topk; ++rk) {
      double best = -1.0;
      int bi = 0x7fffffff;
#pragma unroll
      for (int m = 0; m < MZ; ++m)
        if (z[m] > best) { best = z[m]; bi = lane + 32 * m; }
      seg_argmax(best, bi, 32);
      if (lane == 0) emit(a, l, n0 + r, rk, bi, best);
#pragma unroll
      for (int m = 0; m < MZ; ++m)
        if (lane + 32 * m == bi) z[m] = -2.0;
    }
  }
}

// CTA = one (sequence, block of kRowsPerBlk query rows). Phase 1, one warp
// per query row: scores q.k (ref predictor.py:249, unscaled) held in
// registers, sparsemax threshold by Michelot's fixed point (the support of
// the sorted closed form of ref numkit.py:42-60, tau = (sum_S z - 1)/|S|),
// weights max(z - tau, 0), ctx = w V (dense over T; zero weights are exact
// no-ops), residual + h2 (ref predictor.py:251-252) into smem. Phase 2: the L
// heads for all rows of the block, softmax over K and top-k.
__global__ void __launch_bounds__(32 * kAttnWarps, 1)
attn_heads_kernel(const AttnArgs a) {
  extern __shared__ double smem_d[];
  const int H = a.dm.H, K = a.dm.K;
  const int H3 = 3 * H;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int TS = a.ts;
  double* s_kT = smem_d;                               // H x TS (transposed keys)
  double* s_v = s_kT + (size_t)H * TS;                 // TS x H (values)
  double* s_res = s_v + (size_t)H * TS;                // kRowsPerBlk x kResPitch
  double* s_w = s_res + (size_t)kRowsPerBlk * kResPitch;  // per warp: kMaxLen weights
  double* w_w = s_w + (size_t)wib * kMaxLen;

  const int b = blockIdx.x;
  if (b >= a.blk_off[a.n_seq]) return;
  int lo = 0, hi = a.n_seq - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (a.blk_off[mid] <= b) lo = mid; else hi = mid - 1;
  }
  const int sq = lo;
  const int base = a.seq_off[sq], T = a.seq_off[sq + 1] - base;
  const int r0 = (b - a.blk_off[sq]) * kRowsPerBlk;
  const int r1 = min(T, r0 + kRowsPerBlk);

  unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long tk = clock64();
  auto mark = [&](int i) {
    if (a.prof) {
      const unsigned long long t = clock64();
      ph[i] += t - tk;
      tk = t;
    }
  };

  const bool staged = T <= TS;
  if (staged) {
    for (int i = threadIdx.x; i < H * T; i += blockDim.x) {
      const int j = i / H, c = i % H;
      s_kT[c * TS + j] = a.qkv[(size_t)(base + j) * H3 + H + c];
      s_v[i] = a.qkv[(size_t)(base + j) * H3 + 2 * H + c];
    }
  }
  __syncthreads();
  mark(5);
  const int nz = (T + 31) / 32;  // score registers in use per lane
  for (int r = r0 + wib; r < r1; r += kAttnWarps) {
    const int n = base + r;
    const double* qrow = a.qkv + (size_t)n * H3;
    // ---- scores: lane owns columns j = lane + 32 m
    double z[kMaxZ];
#pragma unroll
    for (int m = 0; m < kMaxZ; ++m) z[m] = 0.0;
    for (int c = 0; c < H; ++c) {
      const double qc = qrow[c];  // uniform address: broadcast
#pragma unroll
      for (int m = 0; m < kMaxZ; ++m) {
        const int j = lane + 32 * m;
        if (m < nz && j < T) {
          const double kv = staged ? s_kT[c * TS + j] : a.qkv[(size_t)(base + j) * H3 + H + c];
          z[m] = fma(qc, kv, z[m]);
        }
      }
    }
    mark(0);
    // ---- sparsemax threshold (Michelot): S_0 = all, tau_i = (sum_{S_i} z - 1)/|S_i|,
    // S_{i+1} = {z > tau_i}, until the support stops shrinking
    double tsum = 0.0;
#pragma unroll
    for (int m = 0; m < kMaxZ; ++m)
      if (m < nz && lane + 32 * m < T) tsum += z[m];
    tsum = warp_sum(tsum);
    int cnt = T;
    double tau = (tsum - 1.0) / (double)cnt;
    for (int it = 0; it < T; ++it) {
      double ssum = 0.0;
      int c = 0;
#pragma unroll
      for (int m = 0; m < kMaxZ; ++m)
        if (m < nz && lane + 32 * m < T && z[m] > tau) {
          ssum += z[m];
          ++c;
        }
      ssum = warp_sum(ssum);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (c == cnt) break;
      cnt = c;
      tau = (ssum - 1.0) / (double)cnt;
    }
    mark(2);
    // ---- weights -> smem; ctx = w V with lanes over h, four chains over j
#pragma unroll
    for (int m = 0; m < kMaxZ; ++m) {
      const int j = lane + 32 * m;
      if (m < nz && j < T) w_w[j] = fmax(z[m] - tau, 0.0);
    }
    __syncwarp();
    double c0[4] = {0.0, 0.0, 0.0, 0.0}, c1[4] = {0.0, 0.0, 0.0, 0.0};
    const int h0 = lane, h1 = lane + 32;
    int j = 0;
    for (; j + 4 <= T; j += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double wj = w_w[j + u];
        const double* vr = staged ? s_v + (size_t)(j + u) * H
                                  : a.qkv + (size_t)(base + j + u) * H3 + 2 * H;
        if (h0 < H) c0[u] = fma(wj, vr[h0], c0[u]);
        if (h1 < H) c1[u] = fma(wj, vr[h1], c1[u]);
      }
    }
    for (; j < T; ++j) {
      const double wj = w_w[j];
      const double* vr = staged ? s_v + (size_t)j * H : a.qkv + (size_t)(base + j) * H3 + 2 * H;
      if (h0 < H) c0[0] = fma(wj, vr[h0], c0[0]);
      if (h1 < H) c1[0] = fma(wj, vr[h1], c1[0]);
    }
    double* res = s_res + (r - r0) * kResPitch;
    if (h0 < H) res[h0] = ((c0[0] + c0[1]) + (c0[2] + c0[3])) + a.h2[(size_t)n * H + h0];
    if (h1 < H) res[h1] = ((c1[0] + c1[1]) + (c1[2] + c1[3])) + a.h2[(size_t)n * H + h1];
    __syncwarp();
    mark(3);
  }
  __syncthreads();
  // ---- L heads over the block's rows
  const int rows = r1 - r0;
  if (K <= 8) heads_small<8>(a, s_res, rows, base + r0);
  else if (K <= 16) heads_small<16>(a, s_res, rows, base + r0);
  else if (K <= 32) heads_small<32>(a, s_res, rows, base + r0);
  else if (K <= 64) heads_large<2>(a, s_res, rows, base + r0);
  else if (K <= 128) heads_large<4>(a, s_res, rows, base + r0);
  else if (K <= 256) heads_large<8>(a, s_res, rows, base + r0);
  else heads_large<32>(a, s_res, rows, base + r0);
  mark(4);
  if (a.prof && lane == 0) {
    unsigned long long* pr = a.prof + ((size_t)blockIdx.x * kAttnWarps + wib) * 8;
    for (int i = 0; i < 6; ++i) pr[i] = ph[i];
  }
}


// ---------------------------------------------------------------------------
// Blocked (GEMM-shaped) attention + heads: one CTA per (sequence, BR query
// rows) -- BR = 64 for T <= 128, BR = 32 for T <= 512 -- 256 threads as a
// 16 x 16 grid with register tiles (RT = BR/16 rows per thread), keys and
// values streamed through smem in chunks of 128:
//   S  = Q K^T          (BR x T, RT x 8 tile per thread, 48-long k loop)
//   sparsemax rows      (warp per row, Michelot threshold; weights in place)
//   R  = W V + h2       (BR x H, RT x 3 tile per thread, over V chunks)
//   Z  = R [heads]      (BR x L*K in layer chunks of <= 128 columns)
//   softmax / top-k     (K <= 32: thread per (row, layer); else warp per (row,
//                        layer); K > 128: online max/sum/top-k
//                        state per row across 128-expert slices)
// The arithmetic per element is the same as attn_heads_kernel; only the
// schedule changes (independent accumulators instead of dependent chains).
constexpr int kBT = 128;       // key / logit chunk
constexpr int kQP = 52;        // pitch (doubles) of Q / K / R rows (= 4 mod 16: DMMA
                               // fragment loads are bank-conflict free)
constexpr int kWP = kBT + 4;   // pitch of the staged head-weight rows (= 4 mod 16)
constexpr int kMaxBlockTop = 8;                    // eval_top_k of the blocked path
constexpr int kStatePitch = 2 + 2 * kMaxBlockTop;   // online heads state per row
template <int BR, int TMAX>
__host__ __device__ constexpr int block_smem() {
  return (kBT * kQP + BR * kQP + BR * (TMAX + 1) + BR * kStatePitch) * 8;
}

struct BlockArgs {
  AttnArgs a;
  const double* hwp;  // heads packed (H, L*K): hwp[i][l*K + e] = head_w[l][i][e]
  double* r_out;      // non-null: write R = ctx + h2 (N, H) here and skip the heads
};

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// out[BR x 128] (pitch op) = A[BR x KP] (pitch kQP) * B, B(k, n) = Bt[n * bn + k * bk]
// on the FP64 tensor cores. 8 warps: BR/16 row groups x 128 / (8 * NTW) column
// groups, NTW 8-wide n-tiles per warp; KP = H rounded up to 4 (zero padded).
template <int BR>
__device__ __forceinline__ void block_dmma(const double* __restrict__ sA, const double* __restrict__ sB,
                                           int bn, int bk, int KP, double* __restrict__ out,
                                           int op) {
  constexpr int RG = BR / 16, CG = 8 / RG, NTW = 16 / CG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp % RG) * 16, c0 = (warp / RG) * NTW * 8;
  double acc[2][NTW][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < KP; k0 += 4) {
    const double a0 = sA[(m0 + g) * kQP + k0 + t];
    const double a1 = sA[(m0 + 8 + g) * kQP + k0 + t];
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      const double b = sB[(c0 + j * 8 + g) * bn + (k0 + t) * bk];
      dmma_884(acc[0][j][0], acc[0][j][1], a0, b);
      dmma_884(acc[1][j][0], acc[1][j][1], a1, b);
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      double* o = out + (m0 + i * 8 + g) * op + c0 + j * 8 + 2 * t;
      o[0] = acc[i][j][0];
      o[1] = acc[i][j][1];
    }
}

template <int BR, int TMAX>
__global__ void __launch_bounds__(256, 1)
attn_block_kernel(const BlockArgs ba) {
  constexpr int RT = BR / 16;          // rows per thread in the register tiles
  constexpr int kSP = TMAX + 1;        // pitch of S / Z rows
  constexpr int NZ = TMAX / 32;        // scores per lane in the sparsemax
  const AttnArgs& a = ba.a;
  extern __shared__ double smem_d[];
  const int H = a.dm.H, K = a.dm.K, L = a.dm.L;
  const int H3 = 3 * H;
  double* sK = smem_d;                  // kBT x kQP   key / value chunk, head weights
  double* sQ = sK + kBT * kQP;          // BR x kQP    queries, later residuals
  double* sS = sQ + BR * kQP;           // BR x kSP    scores -> weights -> logits
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int tx = tid & 15, ty = tid >> 4;

  const int b = blockIdx.x;
  if (b >= a.blk_off[a.n_seq]) return;
  int lo = 0, hi = a.n_seq - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (a.blk_off[mid] <= b) lo = mid; else hi = mid - 1;
  }
  const int base = a.seq_off[lo], T = a.seq_off[lo + 1] - base;
  const int r0 = (b - a.blk_off[lo]) * BR;
  const int rows = min(T - r0, BR);

  const int KP = (H + 3) & ~3;  // DMMA k extent (columns H..KP-1 zero)
  for (int i = tid; i < BR * KP; i += 256) {
    const int r = i / KP, c = i % KP;
    sQ[r * kQP + c] = (r < rows && c < H) ? a.qkv[(size_t)(base + r0 + r) * H3 + c] : 0.0;
  }
  // ---- S = Q K^T over key chunks on the FP64 tensor cores (block_dmma)
  for (int kc = 0; kc < T; kc += kBT) {
    const int nk = min(kBT, T - kc);
    for (int i = tid; i < kBT * KP; i += 256) {
      const int j = i / KP, c = i % KP;
      sK[j * kQP + c] = (j < nk && c < H) ? a.qkv[(size_t)(base + kc + j) * H3 + H + c] : 0.0;
    }
    __syncthreads();
    block_dmma<BR>(sQ, sK, kQP, 1, KP, sS + kc, kSP);
    __syncthreads();
  }

  // ---- sparsemax per row (warp per row): Michelot threshold, weights in place
  for (int r = wib; r < rows; r += 8) {
    double* srow = sS + r * kSP;
    double z[NZ];
#pragma unroll
    for (int m = 0; m < NZ; ++m) z[m] = (lane + 32 * m < T) ? srow[lane + 32 * m] : 0.0;
    double tsum = 0.0;
#pragma unroll
    for (int m = 0; m < NZ; ++m)
      if (lane + 32 * m < T) tsum += z[m];
    tsum = warp_sum(tsum);
    int cnt = T;
    double tau = (tsum - 1.0) / (double)cnt;
    for (int it = 0; it < T; ++it) {
      double ssum = 0.0;
      int cc = 0;
#pragma unroll
      for (int m = 0; m < NZ; ++m)
        if (lane + 32 * m < T && z[m] > tau) {
          ssum += z[m];
          ++cc;
        }
      ssum = warp_sum(ssum);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cc += __shfl_xor_sync(0xffffffffu, cc, o);
      if (cc == cnt) break;
      cnt = cc;
      tau = (ssum - 1.0) / (double)cnt;
    }
#pragma unroll
    for (int m = 0; m < NZ; ++m) {
      const int j = lane + 32 * m;
      if (j < TMAX) srow[j] = (j < T) ? fmax(z[m] - tau, 0.0) : 0.0;
    }
  }
  __syncthreads();

  // ---- R = W V + h2 over value chunks: rows ty*RT + i, columns tx + 16 m (m < 3)
  {
    double acc[RT][3];
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int m = 0; m < 3; ++m) acc[i][m] = 0.0;
    double* sV = sK;  // kBT x 48
    for (int kc = 0; kc < T; kc += kBT) {
      const int nk = min(kBT, T - kc);
      for (int i = tid; i < nk * H; i += 256) {
        const int j = i / H, c = i % H;
        sV[j * 48 + c] = a.qkv[(size_t)(base + kc + j) * H3 + 2 * H + c];
      }
      __syncthreads();
      for (int j = 0; j < nk; ++j) {
        double w[RT], v[3];
#pragma unroll
        for (int i = 0; i < RT; ++i) w[i] = sS[(ty * RT + i) * kSP + kc + j];
#pragma unroll
        for (int m = 0; m < 3; ++m) v[m] = (tx + 16 * m < H) ? sV[j * 48 + tx + 16 * m] : 0.0;
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
          for (int m = 0; m < 3; ++m) acc[i][m] = fma(w[i], v[m], acc[i][m]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      const int r = ty * RT + i;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int c = tx + 16 * m;
        if (r < rows && c < H) {
          const double v = acc[i][m] + a.h2[(size_t)(base + r0 + r) * H + c];
          if (ba.r_out) ba.r_out[(size_t)(base + r0 + r) * H + c] = v;
          else sQ[r * kQP + c] = v;
        }
      }
    }
  }
  if (ba.r_out) return;  // heads in heads_dmma_kernel
  __syncthreads();

  // ---- heads. Logit columns in chunks of <= kBT: whole layers when K <= kBT
  // (lpc layers per chunk), else kBT-expert slices of one layer with an
  // online (max, sum, top-k) state per row carried across the slices.
  const int LK = L * K;
  const int lpc = K <= kBT ? kBT / K : 1;             // layers per chunk
  const int cpl = K <= kBT ? 1 : (K + kBT - 1) / kBT;  // chunks per layer
  double* st = sS + BR * kSP;                          // BR x kStatePitch online state
  for (int l0 = 0; l0 < L; l0 += lpc) {
    const int nl = min(lpc, L - l0);
    for (int ch = 0; ch < cpl; ++ch) {
      const int c0 = ch * kBT;
      const int ncol = K <= kBT ? nl * K : min(kBT, K - c0);
      // Z = R hw[:, col0 : col0 + ncol]: rows ty*4+i, columns tx + 16 m (m < 8);
      // the (H x ncol) weight slice is staged in the (dead) key buffer
      {
        const double* W = ba.hwp + (size_t)l0 * K + c0;
        double* sW = sK;  // KP x kWP (rows H..KP-1 zero)
        for (int i = tid; i < KP * kBT; i += 256) {
          const int c = i / kBT, j = i % kBT;
          sW[c * kWP + j] = (j < ncol && c < H) ? __ldg(W + (size_t)c * LK + j) : 0.0;
        }
        __syncthreads();
        block_dmma<BR>(sQ, sW, 1, kWP, KP, sS, kSP);
      }
      __syncthreads();
      if (K <= 32) {
        // small K: thread per (row, layer), the row's K logits in place in smem
        for (int pr = tid; pr < rows * nl; pr += 256) {
          const int r = pr / nl, l = l0 + pr % nl;
          double* z = sS + r * kSP + (l - l0) * K;
          const double* hb = a.hb + (size_t)l * K;
          double zmax = -INFINITY;
          for (int e = 0; e < K; ++e) {
            z[e] += hb[e];
            zmax = fmax(zmax, z[e]);
          }
          double ssum = 0.0;
          for (int e = 0; e < K; ++e) {
            z[e] = exp(z[e] - zmax);
            ssum += z[e];
          }
          for (int e = 0; e < K; ++e) z[e] = z[e] / ssum;
          for (int rk = 0; rk < a.topk; ++rk) {
            double best = -1.0;
            int bi = 0;
            for (int e = 0; e < K; ++e)
              if (z[e] > best) { best = z[e]; bi = e; }
            emit(a, l, base + r0 + r, rk, bi, best);
            z[bi] = -2.0;
          }
        }
        __syncthreads();
        continue;
      }
      if (K <= kBT) {
        // 32 < K <= 128: eight lanes per (row, layer), 16 logits per lane, four
        // pairs per warp in flight (a warp per pair left the fp64 exp /
        // shuffle chains latency-bound at 8 warps per SM)
        const int grp = lane >> 3, gl = lane & 7;
        const int npairs = rows * nl;
        for (int pb = wib * 4; pb < npairs; pb += 32) {
          const int pr = pb + grp;
          const bool valid = pr < npairs;
          const int r = valid ? pr / nl : 0, l = l0 + (valid ? pr % nl : 0);
          const double* zr = sS + r * kSP + (l - l0) * K;
          const double* hb = a.hb + (size_t)l * K;
          double p[16];
          double zmax = -INFINITY;
#pragma unroll
          for (int m = 0; m < 16; ++m) {
            const int e = gl + 8 * m;
            p[m] = (valid && e < K) ? zr[e] + hb[e] : -INFINITY;
            zmax = fmax(zmax, p[m]);
          }
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
          double ssum = 0.0;
#pragma unroll
          for (int m = 0; m < 16; ++m) {
            p[m] = (valid && gl + 8 * m < K) ? exp(p[m] - zmax) : 0.0;
            ssum += p[m];
          }
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
#pragma unroll
          for (int m = 0; m < 16; ++m) p[m] = (valid && gl + 8 * m < K) ? p[m] / ssum : -2.0;
          for (int rk = 0; rk < a.topk; ++rk) {
            double best = -1.0;
            int bi = 0x7fffffff;
#pragma unroll
            for (int m = 0; m < 16; ++m)  // ascending expert ids: first max = lowest id
              if (p[m] > best) { best = p[m]; bi = gl + 8 * m; }
            seg_argmax(best, bi, 8);
            if (valid && gl == 0) emit(a, l, base + r0 + r, rk, bi, best);
#pragma unroll
            for (int m = 0; m < 16; ++m)
              if (gl + 8 * m == bi) p[m] = -2.0;
          }
        }
        __syncthreads();
        continue;
      }
      // K > 128 (one layer, a 128-expert slice per chunk): eight lanes per row,
      // 16 logits per lane, four rows per warp in flight; online state per
      // row st[r] = {max, sum, (logit, id) x topk}, ids ranked by logit
      // (= probability order), ties to the lower index
      {
        const int grp = lane >> 3, gl = lane & 7;
        const int l = l0;
        const double* hb = a.hb + (size_t)l * K + c0;
        for (int pb = wib * 4; pb < rows; pb += 32) {
          const int r = pb + grp;
          const bool valid = r < rows;
          const double* zr = sS + (valid ? r : 0) * kSP;
          double z[16];
          double zmax = -INFINITY;
#pragma unroll
          for (int m = 0; m < 16; ++m) {
            const int e = gl + 8 * m;
            z[m] = (valid && e < ncol) ? zr[e] + hb[e] : -INFINITY;
            zmax = fmax(zmax, z[m]);
          }
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
          double* srow = st + (valid ? r : 0) * kStatePitch;
          const double prevM = (valid && ch > 0) ? srow[0] : -INFINITY;
          const double M = fmax(prevM, zmax);
          double esum = 0.0;
#pragma unroll
          for (int m = 0; m < 16; ++m)
            if (valid && gl + 8 * m < ncol) esum += exp(z[m] - M);
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) esum += __shfl_xor_sync(0xffffffffu, esum, o);
          const double S = (valid && ch > 0) ? srow[1] * exp(prevM - M) + esum : esum;
          for (int rk = 0; rk < a.topk; ++rk) {
            double best = -INFINITY;
            int bi = 0x7fffffff;
#pragma unroll
            for (int m = 0; m < 16; ++m)
              if (gl + 8 * m < ncol && z[m] > best) { best = z[m]; bi = gl + 8 * m; }
            seg_argmax(best, bi, 8);
#pragma unroll
            for (int m = 0; m < 16; ++m)
              if (gl + 8 * m == bi) z[m] = -INFINITY;
            if (valid && gl == 0 && bi != 0x7fffffff) {
              // insert (best, c0 + bi) into the ranked list (earlier slices
              // hold lower ids, so equal logits keep the earlier entry first)
              double* lst = srow + 2;
              const int n_have = ch > 0 ? a.topk : rk;
              int pos = n_have;
              while (pos > 0 && lst[2 * (pos - 1)] < best) --pos;
              if (pos < a.topk) {
                for (int q = min(n_have, a.topk - 1); q > pos; --q) {
                  lst[2 * q] = lst[2 * (q - 1)];
                  lst[2 * q + 1] = lst[2 * (q - 1) + 1];
                }
                lst[2 * pos] = best;
                lst[2 * pos + 1] = (double)(c0 + bi);
              }
            }
          }
          if (valid && gl == 0) {
            srow[0] = M;
            srow[1] = S;
            if (ch == cpl - 1)
              for (int rk = 0; rk < a.topk; ++rk)
                emit(a, l, base + r0 + r, rk, (int)srow[2 + 2 * rk + 1],
                     exp(srow[2 + 2 * rk] - M) / S);
          }
        }
      }
      __syncthreads();
    }
  }
}

// ---- heads for 8 <= K <= 128, K % 8 == 0 (ref predictor.py:253-259, numkit.py:28-33,87-93):
// logits Z = R hw + hb for all L layers, softmax over each layer's K experts, top-k with
// ties to the lower index. CTA = 8 warps x 8 tokens; per 128-column chunk of the (H, L*K)
// packed head weights (whole layers: 128 / K layers per chunk) the chunk is staged in
// smem once for the CTA and every warp computes its 8 x 128 logits on the FP64 tensor
// cores (m8n8k4: lane (g, t) holds row g, columns 8j + 2t, 8j + 2t + 1), so each row's K
// logits of a layer sit in the four lanes of its quad and every reduction is two
// shuffles. The softmax divides only the picked probabilities: the top-k runs on
// e = exp(z - max) (division by the positive sum is monotone), and an index below the
// pick whose e is within 1e-15 relative is re-checked by its exact quotient, so a tie
// the division creates still resolves to the lower index as in the reference.
constexpr int kHTok = 64;  // tokens per heads CTA
constexpr int heads_smem_bytes() { return (48 * kWP + 128 + kHTok * kQP) * 8; }

__global__ void __launch_bounds__(256, 2)
heads_dmma_kernel(const double* __restrict__ R, int n_tokens, int H, int L, int K,
                  const double* __restrict__ hwp, const double* __restrict__ hb, int topk,
                  int32_t* __restrict__ ids, double* __restrict__ alpha,
                  float* __restrict__ alpha_f32) {
  extern __shared__ double smem_d[];
  double* sW = smem_d;             // KP x kWP chunk of the packed head weights
  double* sB = sW + 48 * kWP;      // 128 biases of the chunk
  double* sR = sB + 128;           // kHTok x kQP residual rows
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int KP = (H + 3) & ~3;
  const int n0 = blockIdx.x * kHTok;
  const int rows = min(kHTok, n_tokens - n0);
  for (int i = tid; i < kHTok * KP; i += 256) {
    const int r = i / KP, c = i - r * KP;
    sR[r * kQP + c] = (r < rows && c < H) ? R[(size_t)(n0 + r) * H + c] : 0.0;
  }
  const int LK = L * K;
  const int lpc = 128 / K, segs = K / 8;
  const int row = warp * 8 + g;
  const bool valid = row < rows;
  const int n = n0 + row;
  // blockIdx.y: this CTA's share of the 128-column chunks (short CTAs: the
  // compute stream's persistent GEMM grids get their SMs back quickly)
  const int n_chunks = ceil_div(L, lpc);
  const int c_lo = blockIdx.y * n_chunks / gridDim.y, c_hi = (blockIdx.y + 1) * n_chunks / gridDim.y;
  for (int l0 = c_lo * lpc; l0 < min(L, c_hi * lpc); l0 += lpc) {
    const int nl = min(lpc, L - l0), ncol = nl * K;
    __syncthreads();  // the previous chunk's readers are done
    for (int i = tid; i < KP * 128; i += 256) {
      const int c = i >> 7, j = i & 127;
      sW[c * kWP + j] = (j < ncol && c < H) ? __ldg(hwp + (size_t)c * LK + (size_t)l0 * K + j) : 0.0;
    }
    if (tid < 128) sB[tid] = tid < ncol ? __ldg(hb + (size_t)l0 * K + tid) : 0.0;
    __syncthreads();
    double acc[16][2];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = 0.0;
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const double a = sR[(warp * 8 + g) * kQP + k0 + t];
#pragma unroll
      for (int j = 0; j < 16; ++j) dmma_884(acc[j][0], acc[j][1], a, sW[(k0 + t) * kWP + j * 8 + g]);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      acc[j][0] += sB[j * 8 + 2 * t];
      acc[j][1] += sB[j * 8 + 2 * t + 1];
    }
    for (int li = 0; li < nl; ++li) {
      const int j0 = li * segs, j1 = j0 + segs;
      double zmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j >= j0 && j < j1) zmax = fmax(zmax, fmax(acc[j][0], acc[j][1]));
      zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, 1));
      zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, 2));
      // e = exp(z - max) in place (only this layer's columns are touched)
      double ssum = 0.0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j >= j0 && j < j1) {
          acc[j][0] = exp(acc[j][0] - zmax);
          acc[j][1] = exp(acc[j][1] - zmax);
          ssum += acc[j][0] + acc[j][1];
        }
      }
      ssum += __shfl_xor_sync(0xffffffffu, ssum, 1);
      ssum += __shfl_xor_sync(0xffffffffu, ssum, 2);
      const int l = l0 + li;
      for (int rk = 0; rk < topk; ++rk) {
        double best = -1.0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int j = 0; j < 16; ++j)  // local ids ascend with (j, q): first max = lowest id
#pragma unroll
          for (int q = 0; q < 2; ++q)
            if (j >= j0 && j < j1 && acc[j][q] > best) {
              best = acc[j][q];
              bi = (j - j0) * 8 + 2 * t + q;
            }
        seg_argmax(best, bi, 4);
        const double p = best / ssum;
        // a lower id whose e is within rounding of best can divide to the same p
        const double near = best * (1.0 - 1e-15);
        int cand = bi;
#pragma unroll
        for (int j = 0; j < 16; ++j)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int id = (j - j0) * 8 + 2 * t + q;
            if (j >= j0 && j < j1 && acc[j][q] >= near && id < cand && acc[j][q] / ssum == p)
              cand = id;
          }
        cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, 1));
        cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, 2));
        if (valid && t == 0) {
          const size_t at = ((size_t)l * n_tokens + n) * topk + rk;
          ids[at] = cand;
          alpha[at] = p;
          if (alpha_f32) alpha_f32[at] = (float)p;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
#pragma unroll
          for (int q = 0; q < 2; ++q)
            if (j >= j0 && j < j1 && (j - j0) * 8 + 2 * t + q == cand) acc[j][q] = -1.0;
      }
    }
  }
}

}  // namespace hash
}  // namespace sida

using namespace sida;
using namespace sida::hash;

static size_t ws_align(size_t b) { return align_up(b, 256); }
static unsigned long long* g_hash_prof = nullptr;
static size_t g_hash_prof_n = 0;

// Observability: phase cycles of the last attention/heads launch when run with
// SIDA_HASH_PROF=1: out[6] = summed (scores, sort, support, ctx, heads, setup).
extern "C" int sida_debug_hash_prof(unsigned long long* out) {
  SIDA_REQUIRE(g_hash_prof, SIDA_ERR_UNSUPPORTED, "run with SIDA_HASH_PROF=1");
  SIDA_CUDA(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(g_hash_prof_n);
  SIDA_CUDA(cudaMemcpy(h.data(), g_hash_prof, g_hash_prof_n * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < 6; ++i) out[i] = 0;
  for (size_t w = 0; w < g_hash_prof_n / 8; ++w)
    for (int i = 0; i < 6; ++i) out[i] += h[w * 8 + i];
  return SIDA_OK;
}

extern "C" size_t sida_hash_param_count(int d, int cd, int H, int L, int K) {
  const size_t G = 4ull * H;
  return (size_t)d * cd + cd + (size_t)cd * G + (size_t)H * G + G + 2ull * H * G + G +
         3ull * H * H + (size_t)L * H * K + (size_t)L * K;
}

extern "C" size_t sida_hash_tables_count(int vocab, int max_len, int H, int L, int K) {
  return ((size_t)vocab + max_len + 1) * 4 * H + 3ull * H * H + (size_t)H * L * K;
}

struct TablePtrs {
  const double *tokx, *posx, *cx, *wqkv, *hwp;
};

static TablePtrs carve_tables(const double* t, int vocab, int max_len, int H) {
  const size_t G = 4ull * H;
  TablePtrs r;
  r.tokx = t;
  r.posx = t + (size_t)vocab * G;
  r.cx = r.posx + (size_t)max_len * G;
  r.wqkv = r.cx + G;
  r.hwp = r.wqkv + 3ull * H * H;
  return r;
}

// Fold the compress FC and the layer-1 input projection into per-vocabulary
// and per-position tables (see the header comment), and pack [Wq|Wk|Wv].
// tok_emb / pos_emb may be NULL (vocab = max_len = 0) for the embed_fn path.
extern "C" int sida_hash_prepare(const double* params, const uint16_t* tok_emb,
                                 const uint16_t* pos_emb, int vocab, int max_len, int d, int cd,
                                 int H, int L, int K, double* tables, void* stream) {
  SIDA_REQUIRE(H >= 1 && H <= 64 && cd >= 1 && cd <= 64, SIDA_ERR_UNSUPPORTED,
               "predictor dims cd=%d H=%d outside the kernel contract (<= 64)", cd, H);
  SIDA_REQUIRE(params && tables && vocab >= 0 && max_len >= 0, SIDA_ERR_CONTRACT,
               "bad hash_prepare arguments");
  cudaStream_t s = as_stream(stream);
  Dims dm{d, cd, H, L, K};
  ParamPtrs w = carve(params, dm);
  const int G = 4 * H;
  TablePtrs t = carve_tables(tables, vocab, max_len, H);
  if (vocab > 0) {
    project_rows_kernel<<<ceil_div(vocab, 8), 256, 0, s>>>(tok_emb, nullptr, vocab, dm, w.cw,
                                                           nullptr, w.wx1,
                                                           const_cast<double*>(t.tokx));
    SIDA_LAUNCH_CHECK();
  }
  if (max_len > 0) {
    project_rows_kernel<<<ceil_div(max_len, 8), 256, 0, s>>>(pos_emb, nullptr, max_len, dm, w.cw,
                                                             nullptr, w.wx1,
                                                             const_cast<double*>(t.posx));
    SIDA_LAUNCH_CHECK();
  }
  bias_project_kernel<<<ceil_div(G, 128), 128, 0, s>>>(w.cb, w.wx1, cd, G,
                                                       const_cast<double*>(t.cx));
  SIDA_LAUNCH_CHECK();
  for (int l = 0; l < L; ++l)  // heads packed (H, L*K)
    SIDA_CUDA(cudaMemcpy2DAsync(const_cast<double*>(t.hwp) + (size_t)l * K,
                                (size_t)L * K * sizeof(double), w.hw + (size_t)l * H * K,
                                K * sizeof(double), K * sizeof(double), H,
                                cudaMemcpyDeviceToDevice, s));
  for (int m = 0; m < 3; ++m) {  // [Wq | Wk | Wv] as one (H x 3H) matrix
    const double* src = m == 0 ? w.wq : (m == 1 ? w.wk : w.wv);
    SIDA_CUDA(cudaMemcpy2DAsync(const_cast<double*>(t.wqkv) + m * H, 3 * H * sizeof(double), src,
                                H * sizeof(double), H * sizeof(double), H,
                                cudaMemcpyDeviceToDevice, s));
  }
  return SIDA_OK;
}

extern "C" size_t sida_hash_workspace_bytes(int n_tokens, int n_seq, int max_len, int d, int cd,
                                            int H, int L, int K) {
  (void)max_len; (void)d; (void)cd; (void)L; (void)K;
  const size_t n = (size_t)n_tokens;
  return ws_align(n * 4 * H * 8) + 2 * ws_align(n * H * 8) + ws_align(n * 3 * H * 8) +
         ws_align(((size_t)n_seq + 1) * 4) + ws_align((size_t)n_seq * H * 8) + 256;
}

static int lstm_chunk() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SIDA_LSTM_CHUNK");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int MAXH, bool FOLD>
static int launch_lstm(const double* xw, const double* tokx, const double* posx, const double* cx,
                       const int32_t* tokens, const double* wh, const double* b,
                       const int32_t* seq_off, int n_seq, int H, double* h_out, cudaStream_t s,
                       int max_len, double* c_buf) {
  int S = 1;
  if (n_seq >= 4 * kNumSMs) S = 4;
  else if (n_seq >= 2 * kNumSMs) S = 2;
  if (S == 4)
    lstm_kernel<MAXH, 4, FOLD><<<ceil_div(n_seq, 4), 4 * MAXH, 0, s>>>(
        xw, tokx, posx, cx, tokens, wh, b, seq_off, n_seq, H, h_out);
  else if (S == 2)
    lstm_kernel<MAXH, 2, FOLD><<<ceil_div(n_seq, 2), 4 * MAXH, 0, s>>>(
        xw, tokx, posx, cx, tokens, wh, b, seq_off, n_seq, H, h_out);
  else if (H == MAXH && !getenv("SIDA_LSTM_SPLIT")) {
    const int chunk = lstm_chunk() > 0 ? lstm_chunk() : max_len;
    for (int t0 = 0; t0 < max_len; t0 += chunk) {
      if (t0 > 0) count_launch();  // SIDA_LAUNCH_CHECK below counts one launch
      lstm_quad_kernel<MAXH, FOLD><<<n_seq, 4 * MAXH, 0, s>>>(
          xw, tokx, posx, cx, tokens, wh, b, seq_off, n_seq, h_out, t0, t0 + chunk, c_buf);
    }
  }
  else
    lstm_kernel<MAXH, 1, FOLD><<<n_seq, 4 * MAXH, 0, s>>>(xw, tokx, posx, cx, tokens, wh, b,
                                                          seq_off, n_seq, H, h_out);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

template <bool FOLD>
static int lstm_dispatch(const double* xw, const double* tokx, const double* posx,
                         const double* cx, const int32_t* tokens, const double* wh,
                         const double* b, const int32_t* seq_off, int n_seq, int H, double* h_out,
                         cudaStream_t s, int max_len, double* c_buf) {
  if (H <= 16) return launch_lstm<16, FOLD>(xw, tokx, posx, cx, tokens, wh, b, seq_off, n_seq, H, h_out, s, max_len, c_buf);
  if (H <= 32) return launch_lstm<32, FOLD>(xw, tokx, posx, cx, tokens, wh, b, seq_off, n_seq, H, h_out, s, max_len, c_buf);
  if (H <= 48) return launch_lstm<48, FOLD>(xw, tokx, posx, cx, tokens, wh, b, seq_off, n_seq, H, h_out, s, max_len, c_buf);
  return launch_lstm<64, FOLD>(xw, tokx, posx, cx, tokens, wh, b, seq_off, n_seq, H, h_out, s, max_len, c_buf);
}

// C (N x M) = A (N x Kd) @ B (Kd x M), fp64 on the FP64 tensor cores (DMMA
// m8n8k4). CTA = 64 rows x all M (<= 192) columns, 8 warps: warp w owns rows
// 16 (w % 4) .. +15 (two 8-row m-tiles) and n-tiles 12 (w / 4) .. +11, i.e.
// 24 DMMA accumulators (48 doubles) per thread. A and B are staged in shared
// memory zero-padded to k % 4 == 0 and n % 8 == 0, with row strides = 4 mod
// 16 doubles so every fragment load is conflict-free (each 16-lane half hits
// 16 distinct double banks).
constexpr int kDR_Rows = 64;
constexpr int kDR_MaxK = 48, kDR_MaxM = 192;

__device__ __forceinline__ int dr_stride(int v) { return (v + 11) / 16 * 16 + 4; }  // >= v, = 4 mod 16

__global__ void __launch_bounds__(256)
rows_dmma_kernel(const double* __restrict__ A, int n_rows, int Kd, const double* __restrict__ B,
                 int M, double* __restrict__ C) {
  extern __shared__ double smem_d[];
  const int KP = (Kd + 3) & ~3, MP = (M + 7) & ~7;
  const int SA = dr_stride(KP), SB = dr_stride(MP);
  double* s_a = smem_d;                   // kDR_Rows x SA
  double* s_b = smem_d + kDR_Rows * SA;   // KP x SB
  const int r0 = blockIdx.x * kDR_Rows;
  for (int i = threadIdx.x; i < KP * MP; i += blockDim.x) {
    const int k = i / MP, c = i - k * MP;
    s_b[k * SB + c] = (k < Kd && c < M) ? B[(size_t)k * M + c] : 0.0;
  }
  for (int i = threadIdx.x; i < kDR_Rows * KP; i += blockDim.x) {
    const int r = i / KP, k = i - r * KP;
    s_a[r * SA + k] = (r0 + r < n_rows && k < Kd) ? A[(size_t)(r0 + r) * Kd + k] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp & 3) * 16;
  const int nt0 = (warp >> 2) * 12;
  const int n_nt = min(12, max(0, MP / 8 - nt0));
  if (n_nt == 0) return;
  double acc[2][12][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 12; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < KP; k0 += 4) {
    const double a0 = s_a[(m0 + g) * SA + k0 + t];
    const double a1 = s_a[(m0 + 8 + g) * SA + k0 + t];
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      if (j < n_nt) {
        const double b = s_b[(k0 + t) * SB + (nt0 + j) * 8 + g];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[0][j][0]), "+d"(acc[0][j][1])
                     : "d"(a0), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[1][j][0]), "+d"(acc[1][j][1])
                     : "d"(a1), "d"(b));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + m0 + i * 8 + g;
    if (r >= n_rows) continue;
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      if (j >= n_nt) continue;
      const int c = (nt0 + j) * 8 + 2 * t;
      double* dst = C + (size_t)r * M + c;
      if (c + 1 < M && (M & 1) == 0) {
        *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (c < M) dst[0] = acc[i][j][0];
        if (c + 1 < M) dst[1] = acc[i][j][1];
      }
    }
  }
}

// SIDA_HASH_HEADS_SPLIT=0: heads inside attn_block_kernel (A/B switch)
static int heads_split() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SIDA_HASH_HEADS_SPLIT");
    v = e ? atoi(e) : 1;
  }
  return v;
}

// SIDA_HASH_DMMA=0: the CUDA-core fp64 kernel below (A/B switch)
static int use_dmma() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SIDA_HASH_DMMA");
    v = e ? atoi(e) : 1;
  }
  return v;
}

static int rows_gemm(const double* A, int n, int Kd, const double* B, int M, double* C,
                     cudaStream_t s) {
  if (use_dmma() && Kd <= kDR_MaxK && M <= kDR_MaxM) {
    const int KP = (Kd + 3) & ~3, MP = (M + 7) & ~7;
    const int SA = (KP + 11) / 16 * 16 + 4, SB = (MP + 11) / 16 * 16 + 4;
    const size_t smem = ((size_t)kDR_Rows * SA + (size_t)KP * SB) * sizeof(double);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
      SIDA_CUDA(cudaFuncSetAttribute(rows_dmma_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      configured = smem;
    }
    rows_dmma_kernel<<<ceil_div(n, kDR_Rows), 256, smem, s>>>(A, n, Kd, B, M, C);
    SIDA_LAUNCH_CHECK();
    return SIDA_OK;
  }
  SIDA_REQUIRE(M >= 1 && M <= 192, SIDA_ERR_UNSUPPORTED, "rows_gemm width %d", M);
  const size_t smem = ((size_t)Kd * M + (size_t)kRG_Rows * (Kd + 1)) * sizeof(double);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    SIDA_CUDA(cudaFuncSetAttribute(rows_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    configured = smem;
  }
  rows_gemm_kernel<<<ceil_div(n, kRG_Rows), 256, smem, s>>>(A, n, Kd, B, M, C);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

// blk_off[i] = sum_{s < i} ceil(len_s / 32)   (attention CTA -> sequence map)
__global__ void block_offsets_kernel(const int32_t* __restrict__ seq_off, int n_seq, int rpb,
                                     int32_t* __restrict__ blk_off) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int acc = 0;
  for (int i = 0; i < n_seq; ++i) {
    blk_off[i] = acc;
    acc += (seq_off[i + 1] - seq_off[i] + rpb - 1) / rpb;
  }
  blk_off[n_seq] = acc;
}

extern "C" int sida_hash_forward(const double* params, const double* tables, int vocab,
                                 int table_max_len, const double* emb_f64,
                                 const int32_t* tokens, const int32_t* seq_off, int n_seq,
                                 int n_tokens, int max_len, int d, int cd, int H, int L, int K,
                                 int topk, int32_t* ids, double* alpha, float* alpha_f32,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  SIDA_REQUIRE(topk >= 1 && topk <= K, SIDA_ERR_CONTRACT, "eval_top_k=%d out of range for K=%d",
               topk, K);
  SIDA_REQUIRE(n_seq >= 1 && n_tokens >= n_seq, SIDA_ERR_CONTRACT, "empty batch or sequence");
  SIDA_REQUIRE(H >= 1 && H <= 48 && cd >= 1 && cd <= 64, SIDA_ERR_UNSUPPORTED,
               "predictor dims cd=%d H=%d outside the kernel contract (H <= 48)", cd, H);
  SIDA_REQUIRE(max_len <= kMaxLen, SIDA_ERR_UNSUPPORTED, "sequence length %d > %d", max_len,
               kMaxLen);
  SIDA_REQUIRE(K <= kMaxK, SIDA_ERR_UNSUPPORTED, "K=%d > %d", K, kMaxK);
  SIDA_REQUIRE(tables && (emb_f64 || (tokens && vocab > 0 && table_max_len >= max_len)),
               SIDA_ERR_CONTRACT, "hash needs prepared tables and embeddings or tokens");
  SIDA_REQUIRE(workspace_bytes >= sida_hash_workspace_bytes(n_tokens, n_seq, max_len, d, cd, H, L, K),
               SIDA_ERR_CONTRACT, "hash workspace too small");
  cudaStream_t s = as_stream(stream);
  Dims dm{d, cd, H, L, K};
  ParamPtrs w = carve(params, dm);
  TablePtrs tb = carve_tables(tables, emb_f64 ? 0 : vocab, emb_f64 ? 0 : table_max_len, H);
  const int G = 4 * H;
  const size_t n = (size_t)n_tokens;
  char* ws = static_cast<char*>(workspace);
  double* xw = reinterpret_cast<double*>(ws); ws += ws_align(n * G * 8);
  double* h1 = reinterpret_cast<double*>(ws); ws += ws_align(n * H * 8);
  double* h2 = reinterpret_cast<double*>(ws); ws += ws_align(n * H * 8);
  double* qkv = reinterpret_cast<double*>(ws); ws += ws_align(n * 3 * H * 8);
  int32_t* blk_off = reinterpret_cast<int32_t*>(ws); ws += ws_align(((size_t)n_seq + 1) * 4);
  double* c_buf = reinterpret_cast<double*>(ws);

  int st;
  if (emb_f64) {
    project_rows_kernel<<<ceil_div(n_tokens, 8), 256, 0, s>>>(nullptr, emb_f64, n_tokens, dm, w.cw,
                                                              w.cb, w.wx1, xw);
    SIDA_LAUNCH_CHECK();
    st = lstm_dispatch<false>(xw, nullptr, nullptr, nullptr, nullptr, w.wh1, w.b1, seq_off, n_seq,
                              H, h1, s, max_len, c_buf);
  } else {
    st = lstm_dispatch<true>(nullptr, tb.tokx, tb.posx, tb.cx, tokens, w.wh1, w.b1, seq_off,
                             n_seq, H, h1, s, max_len, c_buf);
  }
  if (st) return st;
  if ((st = rows_gemm(h1, n_tokens, H, w.wx2, G, xw, s))) return st;
  if ((st = lstm_dispatch<false>(xw, nullptr, nullptr, nullptr, nullptr, w.wh2, w.b2, seq_off,
                                 n_seq, H, h2, s, max_len, c_buf)))
    return st;
  if ((st = rows_gemm(h2, n_tokens, H, tb.wqkv, 3 * H, qkv, s))) return st;
  // blocked path (register-tiled fp64 GEMM shapes, K/V streamed in chunks):
  // 64 query rows per CTA up to T = 128, 32 up to T = 512
  const bool blocked = topk <= kMaxBlockTop && H <= 48 && !getenv("SIDA_HASH_PROF");
  const int rpb = blocked && max_len <= kBT ? 64 : blocked ? 32 : kRowsPerBlk;
  block_offsets_kernel<<<1, 32, 0, s>>>(seq_off, n_seq, rpb, blk_off);
  SIDA_LAUNCH_CHECK();

  AttnArgs a;
  a.qkv = qkv; a.h2 = h2; a.seq_off = seq_off; a.blk_off = blk_off;
  a.n_seq = n_seq; a.n_tokens = n_tokens; a.dm = dm; a.hw = w.hw; a.hb = w.hb; a.topk = topk;
  a.ids = ids; a.alpha = alpha; a.alpha_f32 = alpha_f32;
  a.prof = nullptr;
  const int n_blocks_ub = ceil_div(n_tokens, rpb) + n_seq;
  if (blocked) {
    // K a multiple of 8 up to 128: the heads run in their own kernel (heads_dmma_kernel,
    // 16 warps per SM) on R = ctx + h2 written to the dead xw buffer
    const bool split = K % 8 == 0 && K >= 8 && K <= 128 && H <= 48 && heads_split();
    BlockArgs ba{a, tb.hwp, split ? xw : nullptr};
    if (max_len <= kBT) {
      constexpr int sm = block_smem<64, 128>();
      static bool cfg64 = false;
      if (!cfg64) {
        SIDA_CUDA(cudaFuncSetAttribute(attn_block_kernel<64, 128>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        cfg64 = true;
      }
      attn_block_kernel<64, 128><<<n_blocks_ub, 256, sm, s>>>(ba);
    } else {
      constexpr int sm = block_smem<32, kMaxLen>();
      static bool cfg32 = false;
      if (!cfg32) {
        SIDA_CUDA(cudaFuncSetAttribute(attn_block_kernel<32, kMaxLen>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        cfg32 = true;
      }
      attn_block_kernel<32, kMaxLen><<<n_blocks_ub, 256, sm, s>>>(ba);
    }
    SIDA_LAUNCH_CHECK();
    if (split) {
      constexpr int hs = heads_smem_bytes();
      static bool cfgh = false;
      if (!cfgh) {
        SIDA_CUDA(cudaFuncSetAttribute(heads_dmma_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, hs));
        cfgh = true;
      }
      // split the 128-column chunks over blockIdx.y (SIDA_HEADS_SPLIT_Y, default: one
      // chunk per CTA) so no heads CTA holds an SM for long
      static int split_y = -1;
      if (split_y < 0) {
        const char* e = getenv("SIDA_HEADS_SPLIT_Y");
        split_y = e ? atoi(e) : 0;
      }
      const int n_chunks = ceil_div(L, 128 / K);
      const int gy = split_y > 0 ? std::min(split_y, n_chunks) : n_chunks;
      heads_dmma_kernel<<<dim3(ceil_div(n_tokens, kHTok), gy), 256, hs, s>>>(xw, n_tokens, H, L, K, tb.hwp,
                                                                  w.hb, topk, ids, alpha,
                                                                  alpha_f32);
      SIDA_LAUNCH_CHECK();
    }
    return SIDA_OK;
  }
  if (getenv("SIDA_HASH_PROF")) {
    static unsigned long long* buf = nullptr;
    static size_t cap = 0;
    const size_t need = (size_t)n_blocks_ub * kAttnWarps * 8;
    if (need > cap) {
      if (buf) cudaFree(buf);
      cudaMalloc(&buf, need * sizeof(unsigned long long));
      cap = need;
    }
    cudaMemsetAsync(buf, 0, need * sizeof(unsigned long long), s);
    a.prof = buf;
    g_hash_prof = buf;
    g_hash_prof_n = need;
  }
  // warp-per-row kernel (SIDA_HASH_PROF phase counters, eval_top_k > 8):
  // stage K/V of the sequence in smem when they fit next to the residual and
  // score buffers (227 KB per CTA), else read them from L2
  auto heads_smem = [&](int ts) {
    return ((size_t)2 * H * ts + (size_t)kRowsPerBlk * kResPitch +
            (size_t)kAttnWarps * kMaxLen) * sizeof(double);
  };
  a.ts = heads_smem(max_len) <= 227 * 1024 ? max_len : 0;
  const size_t smem = heads_smem(a.ts);
  static size_t configured = 0;
  if (smem > configured) {
    SIDA_CUDA(cudaFuncSetAttribute(attn_heads_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    configured = smem;
  }
  const int blocks = n_blocks_ub;  // >= sum ceil(len/kRowsPerBlk)
  attn_heads_kernel<<<blocks, 32 * kAttnWarps, smem, s>>>(a);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}
