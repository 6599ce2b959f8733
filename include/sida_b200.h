/*
 * sida_b200.h -- C ABI of the B200-native SiDA serving hot path.
 *
 * One shared library (paper_2310_18859_b200/_sida_b200.so, sm_100a) exports
 * the entry points below. Conventions:
 *   - callers own every buffer; nothing here allocates device memory
 *     (workspace sizes are queried with the *_workspace_bytes helpers);
 *   - every launch takes an explicit stream (a cudaStream_t passed as void*);
 *   - calls are re-entrant across distinct streams and buffers;
 *   - status codes map onto the reference exception taxonomy
 *     (ref pkg/src/sida/errors.py:4-13): no exception crosses the ABI,
 *     the Python mirror raises the matching type. sida_last_error() returns
 *     the calling thread's message for the last non-zero status.
 *
 * Reference interfaces each export replaces are cited per function
 * ("ref" = /root/reference/pkg/src/sida/).
 */
#ifndef SIDA_B200_H
#define SIDA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SIDA_OK = 0,
  SIDA_ERR_CONTRACT = 1,    /* -> ContractError   (ref errors.py:4)  */
  SIDA_ERR_COVERAGE = 2,    /* -> CoverageError   (ref errors.py:8)  */
  SIDA_ERR_UNSERVABLE = 3,  /* -> UnservableError (ref errors.py:12) */
  SIDA_ERR_CUDA = 4,        /* CUDA runtime / launch failure          */
  SIDA_ERR_UNSUPPORTED = 5  /* shape/arch outside the kernel's contract */
};

/* Library identity and the device check (fails unless cc 10.0 / sm_100). */
int sida_abi_version(void);
const char* sida_last_error(void);
/* Number of kernels this library has launched in the process (every entry
 * point counts its own launches; library calls such as cudaMemcpyAsync are
 * not kernels and are not counted). */
unsigned long long sida_launch_count(void);
int sida_device_check(int device);

/* ---------------------------------------------------------------------
 * (1) Hash-function predictor, fp64.
 * Replaces ref predictor.py:373-399 (build_hash_table) over
 * PredictorNet.forward (predictor.py:234-259) + softmax/topk_rows
 * (numkit.py:28-33, 87-93), batched over every sequence of a batch.
 *
 * params: float64, packed in this order (row-major, x@W convention):
 *   compress_w (d,cd) compress_b (cd)
 *   lstm1_wx (cd,4H) lstm1_wh (H,4H) lstm1_b (4H)
 *   lstm2_wx (H,4H)  lstm2_wh (H,4H) lstm2_b (4H)
 *   attn_wq (H,H) attn_wk (H,H) attn_wv (H,H)
 *   head_w (L,H,K) head_b (L,K)
 * tok_emb (vocab,d) / pos_emb (max_len,d): the bf16 embedding tables of the
 *   MoE model (embed = tok_emb[t] + pos_emb[pos], summed in fp64;
 *   ref moe.py:206-218). emb_f64 (n_tokens, d), optional, replaces the
 *   tables for a caller-supplied embed_fn (ref predictor.py:377).
 * tokens: int32 (n_tokens), seq_off: int32 (n_seq+1) exclusive offsets.
 * Outputs, global-token layout (L, n_tokens, topk) (ref moe.py:14-16):
 *   ids int32, alpha float64 (softmax probability at the id, not
 *   renormalised), alpha_f32 optional float32 copy for the FFN epilogue.
 * ------------------------------------------------------------------- */
size_t sida_hash_param_count(int d, int cd, int H, int L, int K);

/* Per-model folding tables (float64, sida_hash_tables_count doubles): the
 * compress FC and layer-1 input projection are linear in the embedding, so
 * TX = (tok_emb Wc) Wx1 (vocab x 4H), PX = (pos_emb Wc) Wx1 (max_len x 4H),
 * cX = bc Wx1, plus [Wq|Wk|Wv] packed (H x 3H) and the heads packed (H x L*K). tok_emb/pos_emb may be NULL
 * with vocab = max_len = 0 (caller-embedding path). Run once per model. */
size_t sida_hash_tables_count(int vocab, int max_len, int H, int L, int K);
int sida_hash_prepare(const double* params, const uint16_t* tok_emb, const uint16_t* pos_emb,
                      int vocab, int max_len, int d, int cd, int H, int L, int K, double* tables,
                      void* stream);

size_t sida_hash_workspace_bytes(int n_tokens, int n_seq, int max_len, int d, int cd, int H,
                                 int L, int K);
/* tables/vocab/table_max_len: from sida_hash_prepare. emb_f64 (n_tokens, d),
 * optional: caller-supplied embeddings (ref predictor.py:377 embed_fn) instead
 * of tokens. Requires H <= 48, cd <= 64, max_len <= 512, K <= 1024. */
int sida_hash_forward(const double* params, const double* tables, int vocab, int table_max_len,
                      const double* emb_f64, const int32_t* tokens, const int32_t* seq_off,
                      int n_seq, int n_tokens, int max_len, int d, int cd, int H, int L, int K,
                      int topk, int32_t* ids, double* alpha, float* alpha_f32, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Observability: summed per-warp cycles of the last hash attention launch by
 * phase (scores, sort, support, ctx, heads, setup) when run with
 * SIDA_HASH_PROF=1. Synchronises the device. */
int sida_debug_hash_prof(unsigned long long* out);

/* ---------------------------------------------------------------------
 * (3) Token permute + histogram (SURVEY §8(a) A13 contract), all layers.
 * ids: int32 (L, n_rows) with n_rows = n_tokens*k, row = token*k + rank.
 * Outputs per layer: hist (L,K), off (L,K+1), perm (L,n_rows) stable by
 * row within expert, inv (L,n_rows) with inv[perm[p]] = p; alpha_perm
 * (optional, L x n_rows float32) = alpha_rows[perm[p]]. err_flag (int32,
 * set to 1 when an id lies outside [0, K), never cleared by the call: a
 * sticky flag the caller zeroes once and reads at its next synchronisation
 * point -> ContractError).
 * Replaces the implicit grouping of ref moe.py:253-256 (w1[ids] gather).
 * ------------------------------------------------------------------- */
size_t sida_permute_workspace_bytes(int n_layers, int n_rows, int num_experts);
int sida_permute_hist(const int32_t* ids, int n_layers, int n_rows, int num_experts,
                      const float* alpha_rows, int32_t* hist, int32_t* off, int32_t* perm,
                      int32_t* inv, float* alpha_perm, int32_t* err_flag, void* workspace,
                      size_t workspace_bytes, void* stream);

/* x_perm[p, :] = bf16(x[perm[p] / k, :]), x float32 (n_tokens, d), 128-bit
 * coalesced. (The row gather half of A13.) */
int sida_gather_rows_bf16(const float* x, const int32_t* perm, int n_rows, int k, int d,
                          uint16_t* x_perm, void* stream);

/* ---------------------------------------------------------------------
 * (4) Expert FFN over permuted rows, bf16 tcgen05/TMEM/TMA grouped GEMM.
 * Replaces ref moe.py:235-262 (moe_apply): per expert e,
 *   f = relu(X_e W1_e + b1_e) W2_e + b2_e, out[row_map[p]] = alpha[p]*f (+ resid)
 * Weights live in HBM slots of one arena (slot stride slot_stride bytes):
 *   [0, h*d*2)        W1^T  (h, d) bf16, K-major
 *   [w2_off, +d*h*2)  W2^T  (d, h) bf16, K-major,  w2_off = h*d*2
 *   [b1_off, +h*2)    b1 (h) bf16,                 b1_off = 2*h*d*2
 *   [b2_off, +d*2)    b2 (d) bf16,                 b2_off = b1_off + h*2
 * expert_slot (K) int32 maps expert -> slot (-1 = not resident: such an
 * expert must have no rows or the call fails with SIDA_ERR_CONTRACT on the
 * device-side check flag). expert_list (n_list, optional) restricts the
 * launch to a subset of experts (layers whose working set exceeds the budget
 * run in waves).
 * row_map (n_rows, optional; identity if NULL): output row of permuted row p.
 * alpha (n_rows, optional; 1 if NULL), resid (optional, indexed like out).
 * out: float32, row stride d; out_bf16 (optional): the same rows rounded to
 * bf16 (the next layer's GEMM input, saving a conversion pass).
 * hidden: bf16 workspace (n_rows, h).
 * Requires d % 64 == 0, h % 64 == 0.
 * ------------------------------------------------------------------- */
size_t sida_slot_bytes(int d, int h);
int sida_grouped_ffn_bf16(const uint16_t* x_perm, int n_rows, int d, int h, const int32_t* off,
                          int num_experts, const int32_t* expert_slot, const int32_t* expert_list,
                          int n_list, const void* arena, size_t slot_stride, int n_slots,
                          const int32_t* row_map, const float* alpha, const float* resid,
                          float* out, uint16_t* out_bf16, uint16_t* hidden, int32_t* err_flag,
                          void* stream);

/* Observability: per-CTA cycle counters of the last sida_grouped_ffn_bf16
 * call when the process runs with SIDA_GEMM_PROF=1 (producer wait, MMA wait
 * on epilogue / on TMA, MMA loop, epilogue wait, epilogue loop, tiles, -,
 * then %globaltimer ns at entry, past the PDL wait, at exit).
 * out: uint64 [2 GEMMs][148 CTAs][12]. Synchronises the device. */
int sida_debug_gemm_prof(unsigned long long* out);
/* Observability: collect the counters above from now on (on = 1) or stop. */
int sida_set_gemm_prof(int on);

/* Expert-FFN tile family for sida_grouped_ffn_bf16: -1 auto (token-N for both
 * GEMMs when d, h % 256 == 0, else token-M), 0 token-M
 * tiles for both GEMMs (128/256 token rows x BN features), 1 token-N tiles
 * for both (swap-AB: 256 features x 16..256 token rows in steps of 16),
 * 2 token-M GEMM1 + token-N GEMM2, 3 token-N GEMM1 + token-M GEMM2,
 * (4, a per-token-tile fused kernel, was retired: contract error), 5 both GEMMs in
 * ONE persistent launch with the hidden rows handed from GEMM1 to GEMM2
 * through L2 (token-N tiles of up to 320 rows, d % 256 == 0, h % 1024 == 0;
 * auto mode runs it for such shapes only with SIDA_XFFN=1).
 * The one-launch path keeps a small per-(device, stream) state buffer
 * (epoch-tagged m-tile flags) allocated on its first call, which therefore
 * must not happen inside a CUDA-graph capture.
 * Process-wide; the initial value comes from SIDA_FFN_SWAP.
 * sida_get_ffn_tiles returns the current mode. */
int sida_set_ffn_tiles(int mode);
int sida_get_ffn_tiles(void);

/* Fused mixing-attention core (ref moe.py:220-233 without the projections):
 * ctx = softmax(q k^T / sqrt(d)) v per sequence, single head, non-causal, on
 * tcgen05 (scores and P.V in TMEM, softmax in registers). qkv bf16
 * (n_tokens, 3d) = [q | k | v]; seq_off int32 (n_seq + 1) device offsets;
 * every sequence <= 512 tokens (max_len), d % 64 == 0; ctx bf16 (n_tokens, d).
 * Up to 256 tokens P = exp(S - max) goes through shared memory; up to 512 it
 * stays in TMEM over the consumed scores and C = P V reads A from TMEM. */
int sida_attention_core(const uint16_t* qkv, const int32_t* seq_off, int n_seq, int n_tokens,
                        int max_len, int d, uint16_t* ctx, void* stream);

/* Embedding and classifier head (the ends of the forward, so a serving step
 * launches only this library's kernels):
 *  - sida_embed: x[t] = tok_emb[tokens[t]] + pos_emb[t - seq_off[s]] for token t
 *    of sequence s (ref moe.py:206-218); tables bf16 (vocab, d) / (max_len, d);
 *    x float32 (n_tokens, d) and its bf16 copy xb; d % 8 == 0;
 *  - sida_pool_classify: logits (n_seq, n_cls) float32 = mean of each
 *    sequence's rows of x @ wc (float32 (d, n_cls)) (ref moe.py:264-266). */
int sida_embed(const int32_t* tokens, const int32_t* seq_off, int n_seq, int n_tokens,
               const uint16_t* tok_emb, const uint16_t* pos_emb, int d, float* x, uint16_t* xb,
               void* stream);
int sida_pool_classify(const float* x, const int32_t* seq_off, int n_seq, int d, const float* wc,
                       int n_cls, float* logits, void* stream);

/* Mixing-attention output projection (ref moe.py:232-233) on the same
 * tcgen05 GEMM, residual fused: out[t] = resid[t] + ctx[t] W_o (fp32), and,
 * for k >= 1, the next FFN's expert-sorted input x_perm[inv[t*k + r]] =
 * bf16(out[t]) for r < k (k <= 4), i.e. the row gather of sida_gather_rows_bf16
 * folded into the epilogue. ctx bf16 (n_rows, d); wo_t = W_o^T (d, d) bf16
 * K-major followed by d zero bf16, sida_out_proj_bytes(d) bytes; d % 64 == 0. */
size_t sida_out_proj_bytes(int d);
int sida_out_proj_scatter(const uint16_t* ctx, int n_rows, int d, const void* wo_t,
                          const float* resid, float* out, const int32_t* inv, int k,
                          uint16_t* x_perm, int32_t* err_flag, void* stream);

/* Dense bf16 linear layer on the same tcgen05 GEMM (used for the mixing
 * attention's fused QKV projection, ref moe.py:225-227): out (n_rows, n) bf16
 * = x (n_rows, k) bf16 @ W + b, with w_t = W^T (n, k) bf16 K-major followed by
 * b (n) bf16, sida_linear_bytes(k, n) bytes; k, n multiples of 64. */
size_t sida_linear_bytes(int k, int n);
int sida_linear_bf16(const uint16_t* x, int n_rows, int k, int n, const void* w_t, uint16_t* out,
                     int32_t* err_flag, void* stream);

/* fp32 FMA check path: same contraction with float32 weights in the
 * reference layout w1 (K,d,h), b1 (K,h), w2 (K,h,d), b2 (K,d); x_perm
 * float32; hidden float32 workspace (n_rows, h). */
int sida_grouped_ffn_f32(const float* x_perm, int n_rows, int d, int h, const int32_t* off,
                         int num_experts, const float* w1, const float* b1, const float* w2,
                         const float* b2, const int32_t* row_map, const float* alpha,
                         const float* resid, float* out, float* hidden, void* stream);

/* Expert parallelism: regroup received bf16 rows
 * (dst[p] = src[idx[p]]) and combine expert outputs returned in the source
 * rank's permuted order: out[t] = resid[t] + sum_r alpha_perm[p] y_perm[p],
 * p = inv[t*k + r], ranks in order; out_bf16 optional. */
int sida_gather_bf16_rows(const uint16_t* src, const int32_t* idx, int n_rows, int d,
                          uint16_t* dst, void* stream);
int sida_unpermute_combine(const uint16_t* y_perm, const int32_t* inv, const float* alpha_perm,
                           const float* resid, int n_tokens, int k, int d, float* out,
                           uint16_t* out_bf16, void* stream);
/* The same combine for any row placement: out[t] = resid[t] + sum_r
 * alpha_rows[t*k + r] y[map[t*k + r]] (alpha in row order), e.g. the
 * expert-parallel NCCL path's chunk-major dispatch order. */
int sida_map_combine(const uint16_t* y, const int32_t* map, const float* alpha_rows,
                     const float* resid, int n_tokens, int k, int d, float* out,
                     uint16_t* out_bf16, void* stream);

/* Expert parallelism over peer memory: the dispatch and
 * return all-to-alls folded into the epilogues that produce the rows.
 * Destinations are encoded v = rank * peer_stride + row; peers (device array
 * of world pointers) are the ranks' bf16 buffers, mapped with
 * sida_ipc_open (NVLink peer mappings on a multi-GPU box).
 *  - sida_out_proj_scatter_peer: as sida_out_proj_scatter, but the bf16 copy
 *    of token t (rank r) goes to the owner's expert-major receive buffer at
 *    map[t*k + r];
 *  - sida_grouped_ffn_bf16_peer: the owner's grouped FFN over its received
 *    rows (off/expert_slot over its num_experts local experts), each output
 *    row (bf16, no alpha / residual) written back to the source rank's buffer
 *    at row_map[j];
 *  - sida_peer_signal / sida_peer_wait: stream-ordered release/acquire flags
 *    (flags_q[me] = epoch on every peer q; wait for flags[0..world) >= epoch);
 *  - sida_segment_map: out[i] = seg_val[b] + p - seg_start[b], p = index[i]
 *    (or i), b the segment of p -- builds the destination maps on the device;
 *  - sida_ipc_handle / sida_ipc_open / sida_ipc_close: CUDA IPC of the
 *    allocation holding a device pointer (sida_ipc_handle_bytes() bytes per
 *    handle, plus the pointer's offset inside the allocation). */
int sida_out_proj_scatter_peer(const uint16_t* ctx, int n_rows, int d, const void* wo_t,
                               const float* resid, float* out, const int32_t* map, int k,
                               uint16_t* const* peers, int peer_stride, int32_t* err_flag,
                               void* stream);
int sida_grouped_ffn_bf16_peer(const uint16_t* x_loc, int n_rows, int d, int h, const int32_t* off,
                               int num_experts, const int32_t* expert_slot, const void* arena,
                               size_t slot_stride, int n_slots, const int32_t* row_map,
                               uint16_t* const* peers, int peer_stride, uint16_t* hidden,
                               int32_t* err_flag, void* stream);
int sida_peer_signal(int32_t* const* peer_flags, int world, int me, int epoch, void* stream);
int sida_peer_wait(const int32_t* flags, int world, int epoch, void* stream);
int sida_segment_map(const int32_t* seg_start, const int32_t* seg_val, int n_seg,
                     const int32_t* index, int n, int32_t* out, void* stream);
size_t sida_ipc_handle_bytes(void);
int sida_ipc_handle(const void* dev_ptr, void* handle_out, size_t* offset_out);
int sida_ipc_open(const void* handle, size_t offset, void** base_out, void** ptr_out);
int sida_ipc_close(void* base);

/* k > 1 combine: out[t] = resid[t] + sum_{r=0..k-1} y[t*k + r] (ranks in
 * order, ref moe.py:252-262). */
int sida_combine_ranks(const float* y, const float* resid, int n_tokens, int k, int d, float* out,
                       uint16_t* out_bf16, void* stream);

/* Router-mode selection (the teacher path): probs = softmax(x W_r) per
 * token, ids = the k most probable experts (descending, equal probabilities
 * to the lower index), alpha = probs at ids (not renormalised). Replaces ref
 * moe.py:296-301 (router branch of forward_sequence) with numkit.py:28-33,
 * 87-93; feeds router-mode model_forward (moe.py:408-442), OracleHasher
 * (predictor.py:413-426) and serve_standard (pipeline.py:370-377).
 * x float32 (n_tokens, d); w_r float32 (d, num_experts), num_experts <= 256;
 * probs float32 (n_tokens, num_experts), optional; ids int32 / alpha float64
 * / alpha_f32 float32 (optional), all (n_tokens, k). */
int sida_router_topk(const float* x, int n_tokens, int d, const float* w_r, int num_experts,
                     int k, float* probs, int32_t* ids, double* alpha, float* alpha_f32,
                     void* stream);

/* ---------------------------------------------------------------------
 * Numeric API of the reference on the GPU, fp64, one CTA per row
 * (the drop-in's utility entry points; the hot path fuses the same math).
 *  - sida_softmax_rows_f64: out = exp(z - max) / sum per row of n
 *    (ref numkit.py:28-33; a few ulp from numpy's);
 *  - sida_sparsemax_rows_f64: the sorted closed form of ref numkit.py:42-60,
 *    bit-identical (n <= 8192);
 *  - sida_topk_rows_f64: idx (rows, k) int64 = argsort(-z, stable)[:k]
 *    (ref numkit.py:76-93), bit-identical;
 *  - sida_router_scores_f64: probs (rows, K) = softmax(x_r @ w_r), x (rows, d),
 *    w_r (d, K) (ref moe.py:108-115 per embedding);
 *  - sida_moe_token_f64: out (d) = sum_i alphas_i (relu(x w1_i + b1_i) w2_i + b2_i)
 *    over the m selected experts packed in selection order, w1 (m, d, h),
 *    b1 (m, h), w2 (m, h, d), b2 (m, d); hidden (m, h) workspace
 *    (ref moe.py:118-146, Eq. 1, no residual).
 * ------------------------------------------------------------------- */
int sida_softmax_rows_f64(const double* z, int rows, int n, double* out, void* stream);
int sida_sparsemax_rows_f64(const double* z, int rows, int n, double* out, void* stream);
int sida_topk_rows_f64(const double* z, int rows, int n, int k, int64_t* idx, void* stream);
int sida_router_scores_f64(const double* x, int rows, int d, const double* w_r, int K,
                           double* probs, void* stream);
int sida_moe_token_f64(const double* x, int m, const double* alphas, const double* w1,
                       const double* b1, const double* w2, const double* b2, int d, int h,
                       double* hidden, double* out, void* stream);

/* ---------------------------------------------------------------------
 * (2) Expert streaming: one pinned-host expert image -> one HBM slot on the
 * copy stream, ordered after wait_event (the slot's last reader) and
 * followed by done_event. Replaces the simulated transfer of ref
 * offload.py:207-222 + pipeline.py:141-146,229-254.
 * ------------------------------------------------------------------- */
int sida_expert_copy(void* dst_slot, const void* src_pinned, size_t bytes, void* copy_stream,
                     void* wait_event, void* done_event);

/* n int32 values from host memory into device memory, in order on
 * `stream`, carried in kernel parameter blocks (no copy-engine work: these
 * small rows never queue behind the expert copies). src may be reused as soon
 * as the call returns. */
int sida_poke_i32(int32_t* dst, const int32_t* src, int n, void* stream);

/* bytes from src to dst copied by the SMs on `stream`; either side may be
 * pinned host memory (mapped under UVA). For the per-batch token rows and
 * logits: no copy-engine work, so they never wait behind expert copies. */
int sida_copy_sm(void* dst, const void* src, size_t bytes, void* stream);

/* Pack one expert from the reference layout (float64 w1 (d,h), b1 (h),
 * w2 (h,d), b2 (d)) into the slot image above (host memory, bf16 RNE).
 * dst must hold sida_slot_bytes(d,h) bytes. */
int sida_pack_expert_host(const double* w1, const double* b1, const double* w2, const double* b2,
                          int d, int h, void* dst);


/* ---------------------------------------------------------------------
 * (2) Residency planner (host, native): ref offload.py:118-204 with the
 * budget in whole expert slots. required: uint8 (L, K) bitmap of the experts
 * each layer of the batch needs (ref predictor.py:96-100). fifo_in: resident
 * keys (layer*K + expert) in arrival order. steps (capacity >= L*K*2 +
 * fifo_len): key for a load, -(key+1) for an eviction, in execution order;
 * group_off (L+1) delimits each layer's group; prefetchable (L) per group.
 * Needs no GPU.
 * ------------------------------------------------------------------- */
int sida_plan_placement(const uint8_t* required, int n_layers, int num_experts, int budget_slots,
                        const int32_t* fifo_in, int fifo_len, int32_t* steps, int steps_capacity,
                        int32_t* group_off, uint8_t* prefetchable);

#ifdef __cplusplus
}
#endif
#endif /* SIDA_B200_H */
