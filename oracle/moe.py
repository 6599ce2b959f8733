"""MoE forward restatement (oracle; test infrastructure only).

Restates the forward half of ref `pkg/src/sida/moe.py`: parameter init
(`:158-181`), `embed` (`:206-218`), `attention_mix` (`:220-233`),
`moe_apply` (`:235-262`), `pool_classify` (`:264-266`), the external-table
batch forward `model_forward(mode="external")` (`:408-442`, `:307-318`) and
the router-mode forward (`:296-306`, `model_forward(mode="router")`).
All arithmetic is float64, sequences are processed one at a time (B=1),
exactly like the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .numkit import make_rng, relu, round_bf16, softmax, topk_rows


@dataclass(frozen=True)
class MoEShape:
    """Mirror of ref `MoEConfig` (`moe.py:40-59`); defaults are the ref's."""

    vocab_size: int = 512
    d_model: int = 64
    num_layers: int = 2
    num_experts: int = 32
    expert_hidden: int = 128
    max_seq_len: int = 64
    routing_k: int = 1
    num_classes: int = 4


def init_params(shape: MoEShape, seed: int) -> dict[str, np.ndarray]:
    """Random init in the reference's draw order (ref `moe.py:158-181`):
    normal(0, 1/sqrt(d)) embeddings, normal(0, sqrt(1/d)) attention/router,
    normal(0, sqrt(2/(d+h))) expert matrices, zero expert biases."""
    g = make_rng(seed)
    d, h, ne = shape.d_model, shape.expert_hidden, shape.num_experts
    p: dict[str, np.ndarray] = {}
    p["tok_emb"] = g.normal(0.0, 1.0 / np.sqrt(d), (shape.vocab_size, d))
    p["pos_emb"] = g.normal(0.0, 1.0 / np.sqrt(d), (shape.max_seq_len, d))
    s_dd, s_dh = np.sqrt(1.0 / d), np.sqrt(2.0 / (d + h))
    for layer in range(shape.num_layers):
        pre = f"block{layer}."
        for name in ("wq", "wk", "wv", "wo"):
            p[pre + name] = g.normal(0.0, s_dd, (d, d))
        p[pre + "w_r"] = g.normal(0.0, s_dd, (d, ne))
        p[pre + "w1"] = g.normal(0.0, s_dh, (ne, d, h))
        p[pre + "b1"] = np.zeros((ne, h))
        p[pre + "w2"] = g.normal(0.0, s_dh, (ne, h, d))
        p[pre + "b2"] = np.zeros((ne, d))
    p["wc"] = g.normal(0.0, s_dd, (d, shape.num_classes))
    return p


def bf16_params(params: dict[str, np.ndarray]) -> dict[str, np.ndarray]:
    """The values the bf16 GPU model holds, as float64."""
    return {k: round_bf16(v) for k, v in params.items()}


def expert_bytes_f64(shape: MoEShape) -> int:
    """ref `moe.py:188-191`: (2dh + h + d) float64 words per expert."""
    return (2 * shape.d_model * shape.expert_hidden + shape.expert_hidden + shape.d_model) * 8


def embed(params, shape: MoEShape, tokens) -> np.ndarray:
    """tok_emb[tokens] + pos_emb[:T] with the ref's checks (ref `moe.py:206-218`)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    if tokens.size == 0:
        raise ValueError("empty sequence")
    if tokens.size > shape.max_seq_len:
        raise ValueError("sequence longer than max_seq_len")
    if tokens.min() < 0 or tokens.max() >= shape.vocab_size:
        raise ValueError("token id out of vocabulary")
    return params["tok_emb"][tokens] + params["pos_emb"][: tokens.size]


def attention_mix(params, shape: MoEShape, layer: int, x: np.ndarray) -> np.ndarray:
    """Single-head non-causal mixing, x + softmax(q k^T / sqrt(d)) v W_o
    (ref `moe.py:220-233`)."""
    pre = f"block{layer}."
    q, k, v = x @ params[pre + "wq"], x @ params[pre + "wk"], x @ params[pre + "wv"]
    att = softmax((q @ k.T) / np.sqrt(shape.d_model))
    return x + (att @ v) @ params[pre + "wo"]


def moe_apply(params, layer: int, x: np.ndarray, ids: np.ndarray, alphas: np.ndarray,
              chunk: int = 16) -> np.ndarray:
    """Routed expert FFN with residual (ref `moe.py:235-262`).

    Like the reference, each token's rank-r expert weights are gathered
    (``w1[ids]``) and contracted per token; ranks accumulate in order
    0..k-1 and the residual is added last (`:262`). ``chunk`` bounds the
    gathered (chunk, d, h) weight block; the per-token arithmetic is the
    reference's.
    """
    pre = f"block{layer}."
    w1, b1, w2, b2 = (params[pre + n] for n in ("w1", "b1", "w2", "b2"))
    ids = np.asarray(ids, dtype=np.int64)
    if ids.min() < 0 or ids.max() >= w1.shape[0]:
        raise ValueError("expert index out of range")
    acc = np.zeros_like(x)
    for r in range(ids.shape[1]):
        f_r = np.empty_like(x)
        for s in range(0, x.shape[0], chunk):
            e = ids[s : s + chunk, r]
            hid = relu(np.einsum("td,tdh->th", x[s : s + chunk], w1[e]) + b1[e])
            f_r[s : s + chunk] = np.einsum("th,thd->td", hid, w2[e]) + b2[e]
        acc += alphas[:, r][:, None] * f_r
    return x + acc


def moe_apply_grouped(params, layer: int, x: np.ndarray, ids: np.ndarray,
                      alphas: np.ndarray) -> np.ndarray:
    """Same contraction as :func:`moe_apply`, evaluated expert-by-expert
    (one BLAS GEMM per (rank, expert)); used only to check large GPU layers
    quickly. Ranks still accumulate in order and the residual comes last."""
    pre = f"block{layer}."
    w1, b1, w2, b2 = (params[pre + n] for n in ("w1", "b1", "w2", "b2"))
    ids = np.asarray(ids, dtype=np.int64)
    acc = np.zeros_like(x)
    for r in range(ids.shape[1]):
        f_r = np.empty_like(x)
        for e in np.unique(ids[:, r]):
            rows = np.nonzero(ids[:, r] == e)[0]
            hid = relu(x[rows] @ w1[e] + b1[e])
            f_r[rows] = hid @ w2[e] + b2[e]
        acc += alphas[:, r][:, None] * f_r
    return x + acc


def pool_classify(params, x: np.ndarray) -> np.ndarray:
    """Mean over tokens then the linear head (ref `moe.py:264-266`)."""
    return x.mean(axis=0) @ params["wc"]


def forward_external(params, shape: MoEShape, sequences, ids: np.ndarray,
                     alphas: np.ndarray, return_layers: bool = False, grouped: bool = False):
    """Batch forward with router bypass (ref `moe.py:408-442` external mode).

    ``ids``/``alphas`` are (L, N, k) over the concatenated token axis.
    ``grouped`` evaluates the experts with :func:`moe_apply_grouped` (same
    contraction, one BLAS GEMM per expert) for Switch-sized checks.
    Returns (logits (B, C), and optionally the per-layer (attn_out, moe_out)
    lists per sequence)."""
    moe_fn = moe_apply_grouped if grouped else moe_apply
    logits, trace = [], []
    off = 0
    for tokens in sequences:
        t = len(tokens)
        x = embed(params, shape, tokens)
        per_layer = []
        for layer in range(shape.num_layers):
            if ids.shape[0] <= layer or off + t > ids.shape[1]:
                raise ValueError(f"missing hash entry for layer {layer}")
            xa = attention_mix(params, shape, layer, x)
            x = moe_fn(params, layer, xa, ids[layer, off : off + t],
                       alphas[layer, off : off + t])
            per_layer.append((xa, x))
        logits.append(pool_classify(params, x))
        trace.append(per_layer)
        off += t
    out = np.stack(logits)
    return (out, trace) if return_layers else out


def router_select(params, layer: int, x: np.ndarray, k: int):
    """Teacher routing (ref `moe.py:296-301`): probs = softmax(x @ w_r),
    sel = topk_rows(probs, k), alphas = probs at sel. Returns (sel, alphas, probs)."""
    probs = softmax(x @ params[f"block{layer}.w_r"])
    sel = topk_rows(probs, k)
    return sel, np.take_along_axis(probs, sel, axis=1), probs


def forward_router(params, shape: MoEShape, sequences, k: int | None = None):
    """Router-mode batch forward (ref `moe.py:408-442` with `forward_sequence`
    `:280-306`): per sequence and layer, attention_mix -> router -> moe_apply.
    Returns (logits (B, C), selected (L, N, k), alphas (L, N, k), probs (L, N, K))."""
    k = shape.routing_k if k is None else k
    logits, sel_rows, al_rows, pr_rows = [], [], [], []
    for tokens in sequences:
        x = embed(params, shape, tokens)
        sels, als, prs = [], [], []
        for layer in range(shape.num_layers):
            x = attention_mix(params, shape, layer, x)
            sel, al, pr = router_select(params, layer, x, k)
            x = moe_apply(params, layer, x, sel, al)
            sels.append(sel)
            als.append(al)
            prs.append(pr)
        logits.append(pool_classify(params, x))
        sel_rows.append(np.stack(sels))
        al_rows.append(np.stack(als))
        pr_rows.append(np.stack(prs))
    return (np.stack(logits), np.concatenate(sel_rows, axis=1),
            np.concatenate(al_rows, axis=1), np.concatenate(pr_rows, axis=1))
