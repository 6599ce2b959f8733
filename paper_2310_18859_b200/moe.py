"""B200 MoE model: host mirror of the forward half of ref pkg/src/sida/moe.py.

Same public names as the reference (`MoEConfig`, `SequenceBatch`,
`ActivationTrace`, `MoEModel`, `model_forward`), but the model lives on the
GPU and runs a whole batch per layer instead of one sequence at a time:

  embed          tok_emb[t] + pos_emb[pos] from bf16 tables (ref moe.py:206-218)
  attention_mix  single-head non-causal mixing (ref moe.py:220-233); cuBLAS
                 bf16 via torch for now (SURVEY §8(f) row 1 makes it a kernel)
  moe_apply      the SiDA hot path: permuted-row gather + tcgen05 grouped FFN
                 with the alpha/unpermute/residual epilogue (ref moe.py:235-262)
  pool_classify  per-sequence mean and linear head (ref moe.py:264-266)

Memory layout: the residual stream x is float32
(n_tokens, d); expert weights never live in this object's device memory --
each (layer, expert) is one pinned host "slot image" (W1^T, W2^T, b1, b2 in
bf16, sida_slot_bytes(d, h) bytes) streamed into HBM slots by
``offload.ExpertStore``.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ContractError


# longest sequence the fused attention core serves (csrc/attention.cu)
MAX_ATTN_TOKENS = 512


@dataclass
class MoEConfig:
    """ref moe.py:40-59 (same fields, defaults and validation)."""

    vocab_size: int = 512
    d_model: int = 64
    num_layers: int = 2
    num_experts: int = 32
    expert_hidden: int = 128
    max_seq_len: int = 64
    routing_k: int = 1
    num_classes: int = 4

    def __post_init__(self):
        for name in ("vocab_size", "d_model", "num_layers", "num_experts", "expert_hidden",
                     "max_seq_len", "routing_k", "num_classes"):
            if getattr(self, name) < 1:
                raise ContractError(f"{name} must be >= 1")
        if self.routing_k > self.num_experts:
            raise ContractError("routing_k must not exceed num_experts")


@dataclass
class SequenceBatch:
    """ref moe.py:62-80."""

    batch_id: int
    sequences: list
    labels: list | None = None

    @property
    def lengths(self) -> list[int]:
        return [len(s) for s in self.sequences]

    @property
    def num_tokens(self) -> int:
        return sum(self.lengths)


@dataclass
class ActivationTrace:
    """ref moe.py:83-105 (external mode: probs is None)."""

    lengths: list[int]
    selected: np.ndarray
    alphas: np.ndarray
    probs: np.ndarray | None

    @property
    def num_layers(self) -> int:
        return self.selected.shape[0]

    @property
    def offsets(self) -> list[int]:
        out = [0]
        for n in self.lengths:
            out.append(out[-1] + n)
        return out


class Rng:
    """Deterministic PCG64 stream over SeedSequence(seed), the generator of
    ref numkit.py:172-209, so `MoEModel(cfg, Rng(s))` draws the reference's
    weights bit-for-bit."""

    algorithm = "pcg64"

    def __init__(self, seed: int, _seq: np.random.SeedSequence | None = None):
        self.seed = int(seed)
        self._seq = _seq if _seq is not None else np.random.SeedSequence(self.seed)
        self._gen = np.random.Generator(np.random.PCG64(self._seq))

    def split(self, n: int) -> list["Rng"]:
        return [Rng(self.seed, _seq=c) for c in self._seq.spawn(n)]

    def integers(self, low, high=None, size=None):
        return self._gen.integers(low, high=high, size=size)

    def normal(self, loc=0.0, scale=1.0, size=None):
        return self._gen.normal(loc=loc, scale=scale, size=size)

    def uniform(self, low=0.0, high=1.0, size=None):
        return self._gen.uniform(low=low, high=high, size=size)

    def random(self, size=None):
        return self._gen.random(size=size)

    def choice(self, a, size=None, replace=True, p=None):
        return self._gen.choice(a, size=size, replace=replace, p=p)

    def permutation(self, x):
        return self._gen.permutation(x)


def router_scores(x, w_r) -> np.ndarray:
    """Softmax over the router's per-expert linear scores for one embedding
    (ref moe.py:108-115), fp64 on the GPU (`sida_router_scores_f64`)."""
    from .numkit import check_finite

    x = check_finite(x, "router input")
    w_r = np.asarray(w_r, dtype=np.float64)
    if x.shape[0] != w_r.shape[0]:
        raise ContractError(
            f"dimension mismatch: x has {x.shape[0]}, router expects {w_r.shape[0]}")
    dev = torch.device("cuda", torch.cuda.current_device())
    xd = torch.from_numpy(np.ascontiguousarray(x.reshape(1, -1))).to(dev)
    wd = torch.from_numpy(np.ascontiguousarray(w_r)).to(dev)
    probs = torch.empty((1, w_r.shape[1]), dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().sida_router_scores_f64(xd.data_ptr(), 1, x.shape[0], wd.data_ptr(),
                                                 w_r.shape[1], probs.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream))
    return probs.cpu().numpy()[0]


def moe_layer_forward(x, selected, alphas, experts, eval_counts: np.ndarray | None = None
                      ) -> np.ndarray:
    """Weighted sum of the selected experts' MLP outputs for one embedding
    (ref moe.py:118-146, Eq. 1), with the reference's contract checks: a
    non-empty selection, ids in range, non-negative alphas. Only the selected
    experts are uploaded and evaluated (`sida_moe_token_f64`, fp64);
    ``eval_counts`` records each evaluation. No residual (the layer adds it)."""
    w1, b1, w2, b2 = (np.asarray(a, dtype=np.float64) for a in experts)
    num_experts = w1.shape[0]
    selected = np.asarray(selected, dtype=np.int64)
    alphas = np.asarray(alphas, dtype=np.float64)
    if selected.size == 0:
        raise ContractError("selected expert set is empty")
    if np.any(selected < 0) or np.any(selected >= num_experts):
        raise ContractError("expert index out of range")
    if np.any(alphas < 0):
        raise ContractError("scaling factors must be non-negative")
    x = np.asarray(x, dtype=np.float64)
    d, h = w1.shape[1], w1.shape[2]
    dev = torch.device("cuda", torch.cuda.current_device())

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    sel = selected.reshape(-1)
    xd, ad = up(x.reshape(-1)), up(alphas.reshape(-1))
    w1d, b1d, w2d, b2d = up(w1[sel]), up(b1[sel]), up(w2[sel]), up(b2[sel])
    hid = torch.empty((sel.size, h), dtype=torch.float64, device=dev)
    out = torch.empty(w2.shape[2], dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().sida_moe_token_f64(
        xd.data_ptr(), int(sel.size), ad.data_ptr(), w1d.data_ptr(), b1d.data_ptr(),
        w2d.data_ptr(), b2d.data_ptr(), d, h, hid.data_ptr(), out.data_ptr(),
        torch.cuda.current_stream().cuda_stream))
    if eval_counts is not None:
        for idx in sel:
            eval_counts[idx] += 1
    return out.cpu().numpy()


def to_bf16(a: np.ndarray, device=None) -> torch.Tensor:
    """float64 -> float32 (RNE) -> bfloat16 (RNE): the one rounding recipe the
    GPU model and the parity oracle share (tests/test_oracle_golden.py)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if not a.flags.writeable:  # memory-mapped checkpoint tensors
        a = a.copy()
    t = torch.from_numpy(a).to(torch.float32)
    t = t.to(torch.bfloat16)
    return t if device is None else t.to(device)


def _default_device():
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError("MoEModel needs a CUDA (sm_100a) device")
    return torch.device("cuda", torch.cuda.current_device())


_SEQ_OFF_CACHE: dict = {}


class BatchLayout:
    """A batch's concatenated global token axis on the device (ref moe.py:14-16):
    int32 tokens and the (n_seq + 1) int32 sequence offsets every kernel of
    the forward reads (uniform batches reuse one cached offsets tensor, so a
    steady-state step moves no per-token metadata)."""

    def __init__(self, lengths: list[int], tokens: torch.Tensor, device):
        self.lengths = [int(n) for n in lengths]
        self.n_seq = len(self.lengths)
        self.n_tokens = int(sum(self.lengths))
        self.max_len = max(self.lengths)
        self.uniform = all(n == self.max_len for n in self.lengths)
        off = np.zeros(self.n_seq + 1, dtype=np.int64)
        np.cumsum(self.lengths, out=off[1:])
        self.offsets = off
        self.tokens = tokens  # int32 (n_tokens,) on device
        dev = torch.device(device)
        if self.uniform:
            key = (dev.index if dev.index is not None else torch.cuda.current_device(),
                   self.n_seq, self.max_len)
            t = _SEQ_OFF_CACHE.get(key)
            if t is None:
                if len(_SEQ_OFF_CACHE) >= 64:
                    _SEQ_OFF_CACHE.pop(next(iter(_SEQ_OFF_CACHE)))
                t = torch.from_numpy(off.astype(np.int32)).to(device)
                _SEQ_OFF_CACHE[key] = t
            self.seq_off = t
        else:
            self.seq_off = torch.from_numpy(off.astype(np.int32)).pin_memory().to(
                device, non_blocking=True)

    @classmethod
    def from_batch(cls, model: "MoEModel", batch: SequenceBatch) -> "BatchLayout":
        toks = model.validate_tokens(batch)
        pinned = torch.from_numpy(toks).pin_memory()
        return cls(batch.lengths, pinned.to(model.device, non_blocking=True), model.device)


def reference_init(config: MoEConfig, rng: Rng) -> dict[str, np.ndarray]:
    """Draw the parameters in the order of ref moe.py:158-181."""
    c = config
    d, h, ne = c.d_model, c.expert_hidden, c.num_experts
    p: dict[str, np.ndarray] = {}
    p["tok_emb"] = rng.normal(0.0, 1.0 / np.sqrt(d), (c.vocab_size, d))
    p["pos_emb"] = rng.normal(0.0, 1.0 / np.sqrt(d), (c.max_seq_len, d))
    for layer in range(c.num_layers):
        pre = f"block{layer}."
        for name in ("wq", "wk", "wv", "wo"):
            p[pre + name] = rng.normal(0.0, np.sqrt(1.0 / d), (d, d))
        p[pre + "w_r"] = rng.normal(0.0, np.sqrt(1.0 / d), (d, ne))
        p[pre + "w1"] = rng.normal(0.0, np.sqrt(2.0 / (d + h)), (ne, d, h))
        p[pre + "b1"] = np.zeros((ne, h))
        p[pre + "w2"] = rng.normal(0.0, np.sqrt(2.0 / (d + h)), (ne, h, d))
        p[pre + "b2"] = np.zeros((ne, d))
    p["wc"] = rng.normal(0.0, np.sqrt(1.0 / d), (d, c.num_classes))
    return p


class MoEModel:
    """Embeddings, mixing attention, experts (as pinned slot images), head.

    ``MoEModel(config, rng)`` draws the reference's weights (ref moe.py:158)
    and holds them at bf16; ``MoEModel(config, params=...)`` takes a reference
    parameter dict; ``MoEModel.synthetic(config, seed)`` draws Switch-shaped
    random weights directly on the GPU for shapes whose float64 reference
    init would not fit host RAM (not reference-identical).
    """

    def __init__(self, config: MoEConfig, rng: Rng | None = None, *, params=None, device=None):
        self.config = config
        self.device = torch.device(device) if device is not None else _default_device()
        self.slot_stride = int(_lib.load().sida_slot_bytes(config.d_model, config.expert_hidden))
        self.expert_images = None  # pinned uint8 (L*K, slot_stride)
        if params is None and rng is None:
            rng = Rng(0)
        if params is None:
            params = reference_init(config, rng)
        self._load_params(params)

    # -- construction -----------------------------------------------------------------
    def _alloc_images(self):
        c = self.config
        self.expert_images = torch.empty((c.num_layers * c.num_experts, self.slot_stride),
                                         dtype=torch.uint8).pin_memory()

    def _load_params(self, params):
        c = self.config
        dev = self.device
        self.tok_emb = to_bf16(params["tok_emb"], dev)
        self.pos_emb = to_bf16(params["pos_emb"], dev)
        self.wqkv, self.wo, self.w_r = [], [], []
        for layer in range(c.num_layers):
            pre = f"block{layer}."
            self.wqkv.append(torch.cat([to_bf16(params[pre + n]) for n in ("wq", "wk", "wv")],
                                       dim=1).to(dev))
            self.wo.append(to_bf16(params[pre + "wo"], dev))
            self.w_r.append(to_bf16(params[pre + "w_r"]).float().to(dev))
        self.wc = to_bf16(params["wc"]).float().to(dev)
        self._prepare_out_proj()
        self._alloc_images()
        h = _lib.load()
        for layer in range(c.num_layers):
            pre = f"block{layer}."
            w1, b1 = params[pre + "w1"], params[pre + "b1"]
            w2, b2 = params[pre + "w2"], params[pre + "b2"]
            for e in range(c.num_experts):
                arrs = [np.ascontiguousarray(a[e], dtype=np.float64) for a in (w1, b1, w2, b2)]
                dst = self.expert_images[layer * c.num_experts + e]
                _lib.check(h.sida_pack_expert_host(*(a.ctypes.data for a in arrs), c.d_model,
                                                   c.expert_hidden, dst.data_ptr()))

    def _stream_handle(self) -> int:
        """Raw handle of the current stream of this model's device."""
        return torch.cuda.current_stream(self._dev_index).cuda_stream

    def _prepare_out_proj(self):
        """Per layer the tcgen05 B operands of the mixing attention's two
        projections, each "W^T (K-major) + a zero bias row": [Wq|Wk|Wv]^T for
        the fused QKV GEMM (sida_linear_bf16) and W_o^T for the output
        projection with its fused residual/scatter epilogue
        (sida_out_proj_scatter). The B200 mixing attention needs
        d_model % 64 == 0 (every Switch shape); other widths have no
        attention path (attention_mix raises), the expert FFN still runs."""
        d = self.config.d_model
        self._dev_index = self.device.index if self.device.index is not None else \
            torch.cuda.current_device()
        self._err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.wo_t = self.wqkv_t = None
        if d % 64:
            return
        h = _lib.load()
        nbytes = int(h.sida_out_proj_bytes(d))
        self.wo_t = []
        for w in self.wo:
            buf = torch.zeros(nbytes // 2, dtype=torch.bfloat16, device=self.device)
            buf[: d * d] = w.t().contiguous().view(-1)
            self.wo_t.append(buf)
        qbytes = int(h.sida_linear_bytes(d, 3 * d))
        self.wqkv_t = []
        for w in self.wqkv:
            buf = torch.zeros(qbytes // 2, dtype=torch.bfloat16, device=self.device)
            buf[: 3 * d * d] = w.t().contiguous().view(-1)
            self.wqkv_t.append(buf)

    @classmethod
    def synthetic(cls, config: MoEConfig, seed: int = 0, device=None) -> "MoEModel":
        """Random-init Switch-shaped weights drawn on the GPU (same scales as
        ref moe.py:163-179: N(0,1/sqrt d) embeddings, N(0,sqrt(1/d)) mixing,
        N(0,sqrt(2/(d+h))) experts, zero biases), rounded to bf16."""
        self = cls.__new__(cls)
        self.config = c = config
        self.device = torch.device(device) if device is not None else _default_device()
        self.slot_stride = int(_lib.load().sida_slot_bytes(c.d_model, c.expert_hidden))
        g = torch.Generator(device=self.device)
        g.manual_seed(int(seed))
        d, hh = c.d_model, c.expert_hidden

        def randn(shape, std, dtype=torch.bfloat16):
            return (torch.randn(shape, generator=g, device=self.device, dtype=torch.float32)
                    * std).to(dtype)

        self.tok_emb = randn((c.vocab_size, d), 1.0 / math.sqrt(d))
        self.pos_emb = randn((c.max_seq_len, d), 1.0 / math.sqrt(d))
        self.wqkv = [randn((d, 3 * d), math.sqrt(1.0 / d)) for _ in range(c.num_layers)]
        self.wo = [randn((d, d), math.sqrt(1.0 / d)) for _ in range(c.num_layers)]
        self.w_r = [randn((d, c.num_experts), math.sqrt(1.0 / d)).float()
                    for _ in range(c.num_layers)]
        self.wc = randn((d, c.num_classes), math.sqrt(1.0 / d)).float()
        self._prepare_out_proj()
        self._alloc_images()
        s_dh = math.sqrt(2.0 / (d + hh))
        n_el = 2 * d * hh
        for i in range(c.num_layers * c.num_experts):
            img = torch.zeros(self.slot_stride // 2, dtype=torch.bfloat16, device=self.device)
            img[:n_el] = randn((n_el,), s_dh)
            self.expert_images[i].copy_(img.view(torch.uint8))
        torch.cuda.synchronize(self.device)
        return self

    def reference_params(self) -> dict[str, np.ndarray]:
        """The model's weights as a reference parameter dict (float64 of the
        bf16 values actually served; ref moe.py:158-181 names and layouts),
        e.g. to check a `synthetic` model end to end against the oracle."""
        c = self.config
        d, hh = c.d_model, c.expert_hidden

        def f64(t):
            return t.detach().float().cpu().numpy().astype(np.float64)

        p = {"tok_emb": f64(self.tok_emb), "pos_emb": f64(self.pos_emb), "wc": f64(self.wc)}
        for layer in range(c.num_layers):
            pre = f"block{layer}."
            wq, wk, wv = f64(self.wqkv[layer]).reshape(d, 3, d).transpose(1, 0, 2)
            p[pre + "wq"], p[pre + "wk"], p[pre + "wv"] = wq, wk, wv
            p[pre + "wo"] = f64(self.wo[layer])
            p[pre + "w_r"] = f64(self.w_r[layer])
            imgs = self.expert_images[layer * c.num_experts:(layer + 1) * c.num_experts]
            raw = imgs.view(torch.bfloat16)[:, : 2 * d * hh + hh + d].float().numpy()
            raw = raw.astype(np.float64)
            p[pre + "w1"] = raw[:, : hh * d].reshape(-1, hh, d).transpose(0, 2, 1).copy()
            p[pre + "w2"] = raw[:, hh * d: 2 * hh * d].reshape(-1, d, hh).transpose(0, 2, 1).copy()
            p[pre + "b1"] = raw[:, 2 * hh * d: 2 * hh * d + hh].copy()
            p[pre + "b2"] = raw[:, 2 * hh * d + hh:].copy()
        return p

    # -- parameter bookkeeping (ref moe.py:188-198) ---------------------------------
    def expert_bytes_each(self) -> int:
        """Bytes one expert occupies in an HBM slot (bf16 image)."""
        return self.slot_stride

    def total_expert_bytes(self) -> int:
        return self.expert_bytes_each() * self.config.num_layers * self.config.num_experts

    def non_expert_bytes(self) -> int:
        n = self.tok_emb.numel() + self.pos_emb.numel()
        n += sum(t.numel() for t in self.wqkv) + sum(t.numel() for t in self.wo)
        return 2 * n + 4 * (self.wc.numel() + sum(t.numel() for t in self.w_r))

    def expert_image(self, layer: int, expert: int) -> torch.Tensor:
        return self.expert_images[layer * self.config.num_experts + expert]

    # -- forward pieces -------------------------------------------------------------
    def validate_tokens(self, batch: SequenceBatch) -> np.ndarray:
        """ref moe.py:208-217 checks, for a whole batch; returns int32 tokens."""
        c = self.config
        if not batch.sequences:
            raise ContractError("empty batch")
        for s in batch.sequences:
            n = len(s)
            if n == 0:
                raise ContractError("empty sequence")
            if n > c.max_seq_len:
                raise ContractError(f"sequence length {n} exceeds max_seq_len {c.max_seq_len}")
        toks = np.concatenate([np.asarray(s, dtype=np.int64) for s in batch.sequences])
        if toks.min() < 0 or toks.max() >= c.vocab_size:
            raise ContractError("token id out of vocabulary")
        return toks.astype(np.int32)

    def embed(self, tokens) -> np.ndarray:
        """One sequence's input embeddings, float64 of the bf16 tables
        (ref moe.py:206-218). The GPU hasher recognises this bound method and
        reads the tables on the device instead of calling it."""
        toks = self.validate_tokens(SequenceBatch(0, [tokens])).astype(np.int64)
        te = self.tok_emb.index_select(0, torch.from_numpy(toks).to(self.device)).double()
        return (te + self.pos_emb[: toks.size].double()).cpu().numpy()

    def embed_layout(self, lay: BatchLayout, with_bf16: bool = False):
        """float32 (n_tokens, d): tok_emb[t] + pos_emb[pos] (exact in fp32),
        one sida_embed launch; ``with_bf16`` also returns its bf16 copy (the
        first QKV projection's input) from the same kernel."""
        d = self.config.d_model
        x = torch.empty((lay.n_tokens, d), dtype=torch.float32, device=self.device)
        xb = torch.empty((lay.n_tokens, d), dtype=torch.bfloat16, device=self.device)
        _lib.check(_lib.lib().sida_embed(
            lay.tokens.data_ptr(), lay.seq_off.data_ptr(), lay.n_seq, lay.n_tokens,
            self.tok_emb.data_ptr(), self.pos_emb.data_ptr(), d, x.data_ptr(), xb.data_ptr(),
            self._stream_handle()))
        return (x, xb) if with_bf16 else x

    def attention_mix(self, layer: int, x: torch.Tensor, lay: BatchLayout,
                      xb: torch.Tensor | None = None, scatter=None) -> torch.Tensor:
        """x + softmax(q k^T / sqrt(d)) v W_o per sequence (ref moe.py:220-233),
        three tcgen05 launches: the fused QKV projection (sida_linear_bf16),
        the attention core (sida_attention_core: scores, softmax and P.V
        on chip, sequences of up to 512 tokens) and the output projection
        (sida_out_proj_scatter) with the residual add fused -- given
        ``scatter = (inv, k, x_perm)`` from the layer's hash table it also
        writes the next FFN's expert-sorted bf16 input rows x_perm[inv[t*k+r]]
        (the row gather of ref moe.py:253-256), so the FFN needs no gather
        pass. ``xb`` is x already rounded to bf16 (the embedding kernel or the
        previous layer's FFN epilogue writes it)."""
        d = self.config.d_model
        if self.wo_t is None:
            raise _lib.NativeLibraryError(
                f"the B200 mixing attention needs d_model % 64 == 0 (got {d})")
        if lay.max_len > MAX_ATTN_TOKENS:
            raise _lib.NativeLibraryError(
                f"the fused attention core serves sequences of at most {MAX_ATTN_TOKENS} "
                f"tokens (got {lay.max_len})")
        if xb is None:
            xb = x.to(torch.bfloat16)
        h = _lib.lib()
        sh = self._stream_handle()
        qkv = torch.empty((lay.n_tokens, 3 * d), dtype=torch.bfloat16, device=x.device)
        _lib.check(h.sida_linear_bf16(xb.data_ptr(), lay.n_tokens, d, 3 * d,
                                      self.wqkv_t[layer].data_ptr(), qkv.data_ptr(),
                                      self._err.data_ptr(), sh))
        ctx = torch.empty((lay.n_tokens, d), dtype=torch.bfloat16, device=x.device)
        _lib.check(h.sida_attention_core(qkv.data_ptr(), lay.seq_off.data_ptr(), lay.n_seq,
                                         lay.n_tokens, lay.max_len, d, ctx.data_ptr(), sh))
        return self._out_proj(layer, x, ctx, scatter)

    def _out_proj(self, layer: int, x: torch.Tensor, ctx: torch.Tensor, scatter):
        d = self.config.d_model
        out = torch.empty_like(x)
        if scatter is not None and scatter[0] == "peer":
            # expert parallel: rows go straight to the owners' receive buffers
            _, dmap, k, peers, stride = scatter
            _lib.check(_lib.lib().sida_out_proj_scatter_peer(
                ctx.data_ptr(), ctx.shape[0], d, self.wo_t[layer].data_ptr(), x.data_ptr(),
                out.data_ptr(), dmap.data_ptr(), k, peers.data_ptr(), stride,
                self._err.data_ptr(), self._stream_handle()))
            return out
        inv, k, x_perm = scatter if scatter is not None else (None, 0, None)
        _lib.check(_lib.lib().sida_out_proj_scatter(
            ctx.data_ptr(), ctx.shape[0], d, self.wo_t[layer].data_ptr(), x.data_ptr(),
            out.data_ptr(), _lib.ptr(inv), k, _lib.ptr(x_perm), self._err.data_ptr(),
            self._stream_handle()))
        return out

    def pool_classify(self, x: torch.Tensor, lay: BatchLayout) -> torch.Tensor:
        """(n_seq, C): per-sequence mean then the classifier (ref moe.py:264-266),
        one sida_pool_classify launch."""
        c = self.config
        logits = torch.empty((lay.n_seq, c.num_classes), dtype=torch.float32, device=self.device)
        _lib.check(_lib.lib().sida_pool_classify(x.data_ptr(), lay.seq_off.data_ptr(), lay.n_seq,
                                                 c.d_model, self.wc.data_ptr(), c.num_classes,
                                                 logits.data_ptr(), self._stream_handle()))
        return logits

    def route(self, layer: int, x: torch.Tensor, k: int, stream=None, want_probs: bool = True):
        """Teacher routing on the GPU (ref moe.py:296-301): one fused kernel,
        probs = softmax(x W_r), the k most probable experts (ties to the lower
        index) and their probabilities. Returns (ids int32 (1, N, k), alpha
        float64 (1, N, k), alpha float32 (1, N, k), probs float32 (N, K) or None)."""
        c = self.config
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        n = x.shape[0]
        dev = self.device
        ids = torch.empty((1, n, k), dtype=torch.int32, device=dev)
        alpha = torch.empty((1, n, k), dtype=torch.float64, device=dev)
        alpha32 = torch.empty((1, n, k), dtype=torch.float32, device=dev)
        probs = torch.empty((n, c.num_experts), dtype=torch.float32, device=dev) if want_probs else None
        _lib.check(_lib.lib().sida_router_topk(
            x.data_ptr(), n, c.d_model, self.w_r[layer].data_ptr(), c.num_experts, k,
            _lib.ptr(probs), ids.data_ptr(), alpha.data_ptr(), alpha32.data_ptr(), st.cuda_stream))
        return ids, alpha, alpha32, probs

    def moe_apply_rows(self, layer_tables, x: torch.Tensor, k: int, arena, slot_row: torch.Tensor,
                       expert_list: torch.Tensor | None = None, out: torch.Tensor | None = None,
                       y: torch.Tensor | None = None, stream=None,
                       out_bf16: torch.Tensor | None = None,
                       x_perm: torch.Tensor | None = None) -> torch.Tensor:
        """The SiDA expert FFN for one layer over the whole batch.

        ``layer_tables`` = (off (K+1,), perm (R,), alpha_perm (R,)) of this
        layer from sida_permute_hist; ``slot_row`` (K,) int32 expert -> slot.
        k == 1: out[t] = x[t] + alpha * f(x[t]) written by the GEMM2
        epilogue directly (unpermute + residual fused), plus its bf16 copy in
        ``out_bf16`` when given. k > 1: the epilogue writes alpha_r f_r into
        row t*k+r of ``y`` and sida_combine_ranks adds the ranks in order plus
        the residual (ref moe.py:252-262).
        """
        c = self.config
        h = _lib.lib()
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        sh = st.cuda_stream
        off, perm, alpha_perm = layer_tables
        n_tok = x.shape[0]
        rows = n_tok * k
        hidden = torch.empty((rows, c.expert_hidden), dtype=torch.bfloat16, device=self.device)
        if x_perm is None:  # not produced by the fused output projection: gather
            x_perm = torch.empty((rows, c.d_model), dtype=torch.bfloat16, device=self.device)
            _lib.check(h.sida_gather_rows_bf16(x.data_ptr(), perm.data_ptr(), rows, k, c.d_model,
                                               x_perm.data_ptr(), sh))
        err = arena.err_flag
        n_list = 0 if expert_list is None else int(expert_list.numel())
        if out is None:
            out = torch.empty_like(x)
        if k == 1:
            target, resid = out, x
        else:
            target = y if y is not None else torch.empty((rows, c.d_model), dtype=torch.float32,
                                                         device=self.device)
            resid = None
        args = (x_perm.data_ptr(), rows, c.d_model, c.expert_hidden, off.data_ptr(),
                c.num_experts, slot_row.data_ptr(), _lib.ptr(expert_list), n_list,
                arena.base_ptr, arena.slot_stride, arena.n_slots, perm.data_ptr(),
                alpha_perm.data_ptr(), _lib.ptr(resid), target.data_ptr(),
                _lib.ptr(out_bf16 if k == 1 else None), hidden.data_ptr(), err.data_ptr())
        _lib.check(h.sida_grouped_ffn_bf16(*args, sh))
        return target

    def combine(self, y: torch.Tensor, x: torch.Tensor, k: int, out: torch.Tensor | None = None,
                stream=None, out_bf16: torch.Tensor | None = None) -> torch.Tensor:
        h = _lib.lib()
        st = torch.cuda.current_stream(self.device) if stream is None else stream
        if out is None:
            out = torch.empty_like(x)
        _lib.check(h.sida_combine_ranks(y.data_ptr(), x.data_ptr(), x.shape[0], k,
                                        self.config.d_model, out.data_ptr(), _lib.ptr(out_bf16),
                                        st.cuda_stream))
        return out


def router_forward(model: MoEModel, lay: BatchLayout, ktop: int, store=None, stream=None):
    """Router-mode forward of a whole batch on the device (ref moe.py:280-306
    router branch, per layer: attention_mix -> softmax(x W_r) -> top-k ->
    moe_apply). ``ktop`` >= routing_k experts are selected per token; the
    first routing_k route the token (top-k orders are prefixes of each
    other). Returns device tensors (logits (B, C), ids int32 (L, N, ktop),
    alpha float64 (L, N, ktop), probs float32 (L, N, K))."""
    from .offload import ExpertStore  # local import: offload depends on moe
    from .predictor import DeviceTable

    c = model.config
    st = stream or torch.cuda.current_stream(model.device)
    store = store or ExpertStore.full(model)
    rk = c.routing_k
    n = lay.n_tokens
    ids_all = torch.empty((c.num_layers, n, ktop), dtype=torch.int32, device=model.device)
    al_all = torch.empty((c.num_layers, n, ktop), dtype=torch.float64, device=model.device)
    pr_all = torch.empty((c.num_layers, n, c.num_experts), dtype=torch.float32,
                         device=model.device)
    with torch.cuda.stream(st):
        x = model.embed_layout(lay)
        for layer in range(c.num_layers):
            x = model.attention_mix(layer, x, lay)
            ids, al, al32, pr = model.route(layer, x, ktop, stream=st)
            ids_all[layer].copy_(ids[0])
            al_all[layer].copy_(al[0])
            pr_all[layer].copy_(pr)
            if ktop != rk:
                ids, al, al32 = (t[:, :, :rk].contiguous() for t in (ids, al, al32))
            dt = DeviceTable(ids, al, al32, n, rk)
            dt.permute(c.num_experts, st)
            x = store.run_layer(model, layer, x, dt, stream=st, table_layer=0)
        logits = model.pool_classify(x, lay)
    return logits, ids_all, al_all, pr_all


def model_forward(model: MoEModel, batch: SequenceBatch, mode: str = "router", table=None,
                  timings: dict | None = None, store=None):
    """Forward a whole batch (ref moe.py:408-442); returns (logits numpy
    (B, C), ActivationTrace).

    ``mode="router"``: the teacher routers select the experts on the GPU
    (`sida_router_topk` per layer); the trace holds the selections, their
    probabilities and the full router distributions. ``mode="external"``:
    the hash table's (ids, alphas) replace the routers. Every expert a layer
    needs is made resident in ``store`` (default: a store holding all
    experts) before its layer runs.
    """
    from .offload import ExpertStore  # local import: offload depends on moe

    if mode not in ("router", "external"):
        raise ContractError(f"unknown forward mode {mode!r}")
    if store is None:
        store = ExpertStore.full(model)
    if mode == "router":
        lay = BatchLayout.from_batch(model, batch)
        t0 = time.perf_counter()
        logits, ids, al, pr = router_forward(model, lay, model.config.routing_k, store)
        out = logits.cpu().numpy().astype(np.float64)
        _check_flags(model, store)
        if timings is not None:
            timings["forward"] = timings.get("forward", 0.0) + time.perf_counter() - t0
        trace = ActivationTrace(lengths=batch.lengths, selected=ids.cpu().numpy().astype(np.int64),
                                alphas=al.cpu().numpy(), probs=pr.cpu().numpy().astype(np.float64))
        return out, trace
    if table is None:
        raise ContractError("external mode requires a hash table")
    dev_table = table.on_device(model)
    if dev_table.n_tokens != batch.num_tokens or table.lengths != batch.lengths:
        raise ContractError("hash table does not cover the requested tokens")
    if dev_table.num_layers < model.config.num_layers:
        raise ContractError(f"missing hash entry for (layer {dev_table.num_layers}, token 0)")
    lay = BatchLayout(batch.lengths, dev_table.tokens_for(model, batch), model.device)
    x = model.embed_layout(lay)
    torch.cuda.current_stream(model.device).wait_event(dev_table.ready)
    for layer in range(model.config.num_layers):
        x = model.attention_mix(layer, x, lay)
        x = store.run_layer(model, layer, x, dev_table)
    logits = model.pool_classify(x, lay).cpu().numpy().astype(np.float64)
    _check_flags(model, store, dev_table)
    trace = ActivationTrace(lengths=batch.lengths, selected=table.ids, alphas=table.alphas,
                            probs=None)
    return logits, trace


def _check_flags(model: MoEModel, store, dev_table=None) -> None:
    from .offload import FFN_SLOT_MSG, OUTPROJ_MSG, PERMUTE_MSG, check_device_flags

    check_device_flags([(FFN_SLOT_MSG, store.err_flag), (OUTPROJ_MSG, model._err),
                        (PERMUTE_MSG, dev_table.err if dev_table is not None else None)])
