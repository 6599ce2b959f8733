"""Hash-function predictor restatement (oracle; test infrastructure only).

Restates the inference half of ref `pkg/src/sida/predictor.py`:
parameter init (`:132-164`), the LSTM recurrence (`:174-196`), the forward
(`:234-259`) and `build_hash_table` (`:373-399`). Float64 throughout.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .numkit import make_rng, sigmoid, softmax, sparsemax, topk_rows


@dataclass(frozen=True)
class PredictorShape:
    """Mirror of the inference-relevant fields of ref `PredictorConfig`
    (`predictor.py:41-58`) plus the model dims `PredictorNet` takes."""

    d_model: int
    num_moe_layers: int
    num_experts: int
    compress_dim: int = 24
    lstm_hidden: int = 48


def init_params(shape: PredictorShape, seed: int) -> dict[str, np.ndarray]:
    """Draw order of ref `predictor.py:145-164`: xavier compress, uniform
    +-1/sqrt(H) LSTM matrices with forget-gate bias 1, xavier attention and
    per-layer heads, zero biases."""
    g = make_rng(seed)
    d, cd, hid = shape.d_model, shape.compress_dim, shape.lstm_hidden

    def xavier(fan_in, fan_out, size):
        return g.normal(0.0, np.sqrt(2.0 / (fan_in + fan_out)), size)

    p: dict[str, np.ndarray] = {"compress_w": xavier(d, cd, (d, cd)), "compress_b": np.zeros(cd)}
    bound = 1.0 / np.sqrt(hid)
    for idx, n_in in ((1, cd), (2, hid)):
        p[f"lstm{idx}_wx"] = g.uniform(-bound, bound, (n_in, 4 * hid))
        p[f"lstm{idx}_wh"] = g.uniform(-bound, bound, (hid, 4 * hid))
        bias = np.zeros(4 * hid)
        bias[hid : 2 * hid] = 1.0
        p[f"lstm{idx}_b"] = bias
    for name in ("attn_wq", "attn_wk", "attn_wv"):
        p[name] = xavier(hid, hid, (hid, hid))
    p["head_w"] = xavier(hid, shape.num_experts, (shape.num_moe_layers, hid, shape.num_experts))
    p["head_b"] = np.zeros((shape.num_moe_layers, shape.num_experts))
    return p


def lstm(wx: np.ndarray, wh: np.ndarray, b: np.ndarray, x: np.ndarray) -> np.ndarray:
    """(T, n_in) -> (T, H); zero initial state, gate blocks i|f|g|o,
    c = f*c + i*g, h = o*tanh(c) (ref `predictor.py:174-196`)."""
    hid = wh.shape[0]
    h = np.zeros(hid)
    c = np.zeros(hid)
    out = np.empty((x.shape[0], hid))
    for t in range(x.shape[0]):
        z = x[t] @ wx + h @ wh + b
        i_g = sigmoid(z[:hid])
        f_g = sigmoid(z[hid : 2 * hid])
        g_g = np.tanh(z[2 * hid : 3 * hid])
        o_g = sigmoid(z[3 * hid :])
        c = f_g * c + i_g * g_g
        h = o_g * np.tanh(c)
        out[t] = h
    return out


def forward(params, emb: np.ndarray, return_parts: bool = False):
    """(T, d) embeddings -> (L, T, K) logits (ref `predictor.py:234-259`).

    Note the unscaled q k^T scores (`:249`) and the residual ctx + h2
    (`:252`) ahead of the per-layer heads (`:253`)."""
    emb = np.asarray(emb, dtype=np.float64)
    if emb.shape[0] < 1:
        raise ValueError("empty sequence")
    comp = emb @ params["compress_w"] + params["compress_b"]
    h1 = lstm(params["lstm1_wx"], params["lstm1_wh"], params["lstm1_b"], comp)
    h2 = lstm(params["lstm2_wx"], params["lstm2_wh"], params["lstm2_b"], h1)
    q, k, v = h2 @ params["attn_wq"], h2 @ params["attn_wk"], h2 @ params["attn_wv"]
    w = sparsemax(q @ k.T)
    resid = w @ v + h2
    logits = np.einsum("th,lhk->ltk", resid, params["head_w"]) + params["head_b"][:, None, :]
    if return_parts:
        return logits, dict(comp=comp, h1=h1, h2=h2, weights=w, resid=resid)
    return logits


def build_hash_table(params, sequences, eval_top_k: int, embed_fn):
    """Per sequence: embed -> forward -> softmax over K -> top-k of the
    probabilities; alpha = the (un-renormalised) probability at each id;
    concatenated on the global token axis (ref `predictor.py:373-399`).
    Returns (ids int64 (L, N, k), alphas float64 (L, N, k))."""
    if eval_top_k < 1:
        raise ValueError("eval_top_k must be >= 1")
    ids, alphas = [], []
    for tokens in sequences:
        probs = softmax(forward(params, embed_fn(tokens)))
        sel = topk_rows(probs, eval_top_k)
        ids.append(sel)
        alphas.append(np.take_along_axis(probs, sel, axis=-1))
    return np.concatenate(ids, axis=1), np.concatenate(alphas, axis=1)


def top_gap(params, emb: np.ndarray) -> np.ndarray:
    """Relative gap between the top-1 and top-2 probability per (layer,
    token): the margin an fp64 re-association must stay inside for ids to be
    bit-exact (SURVEY §7 "bit-exact ids")."""
    probs = softmax(forward(params, emb))
    srt = np.sort(probs, axis=-1)
    return (srt[..., -1] - srt[..., -2]) / srt[..., -1]


def oracle_table(probs: np.ndarray, eval_top_k: int):
    """`OracleHasher.build_table` (ref `predictor.py:419-426`): top-k of the
    teacher's router probabilities (L, N, K) -> (ids, alphas) (L, N, k)."""
    L, N, K = probs.shape
    sel = topk_rows(probs.reshape(-1, K), eval_top_k).reshape(L, N, eval_top_k)
    return sel, np.take_along_axis(probs, sel, axis=-1)


def hash_hit_rate(pred_ids: list, teacher_sel: list, k: int) -> float:
    """ref `predictor.py:429-449`: fraction of (layer, token) whose teacher
    top-1 expert is among the first k predicted ids."""
    hits = total = 0
    for ids, sel in zip(pred_ids, teacher_sel):
        top1 = sel[:, :, 0]
        hits += int(np.sum(np.any(ids[:, :, :k] == top1[:, :, None], axis=-1)))
        total += top1.size
    return hits / total
