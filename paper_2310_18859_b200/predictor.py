"""SiDA hash function on the GPU: host mirror of the inference half of
ref pkg/src/sida/predictor.py.

`build_hash_table` keeps the reference signature (ref predictor.py:373) but
runs every sequence of the batch in one fp64 kernel chain
(`sida_hash_forward`) and immediately permutes every layer's (token, rank)
rows by expert (`sida_permute_hist`) on the same stream.
The resulting `ExpertHashTable` is device-resident; its numpy views
(`ids`, `alphas`) are fetched lazily -- boundary (iv) of SURVEY §3.
"""

from __future__ import annotations

import json
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ContractError, CoverageError
from .moe import BatchLayout, MoEModel, Rng, SequenceBatch, router_forward


@dataclass
class PredictorConfig:
    """ref predictor.py:41-58 (training fields kept for API parity)."""

    compress_dim: int = 24
    lstm_hidden: int = 48
    lstm_layers: int = 2
    top_t: int = 30
    lambda_ce: float = 0.005
    lr: float = 5e-5
    batch_size: int = 64
    max_steps: int = 2000

    def __post_init__(self):
        if self.lstm_layers != 2:
            raise ContractError("the predictor trunk is fixed at 2 LSTM layers")
        if self.top_t < 1:
            raise ContractError("top_t must be >= 1")
        if self.lambda_ce < 0:
            raise ContractError("lambda_ce must be >= 0")


PARAM_ORDER = ("compress_w", "compress_b", "lstm1_wx", "lstm1_wh", "lstm1_b", "lstm2_wx",
               "lstm2_wh", "lstm2_b", "attn_wq", "attn_wk", "attn_wv", "head_w", "head_b")


class PredictorNet:
    """Compress FC -> 2-layer LSTM -> sparsemax attention -> residual -> heads
    (ref predictor.py:129-164); parameters float64, packed once on the device
    in the order sida_hash_forward expects (include/sida_b200.h)."""

    def __init__(self, config: PredictorConfig, d_model: int, num_moe_layers: int,
                 num_experts: int, rng: Rng | None = None, *, params=None):
        self.config = config
        self.d_model = d_model
        self.num_moe_layers = num_moe_layers
        self.num_experts = num_experts
        if params is None:
            params = self._init(rng if rng is not None else Rng(0))
        self.params = params
        self._packed = {}

    def _init(self, rng: Rng) -> dict[str, np.ndarray]:
        cd, hid = self.config.compress_dim, self.config.lstm_hidden

        def xavier(n_in, n_out, shape):
            return rng.normal(0.0, np.sqrt(2.0 / (n_in + n_out)), shape)

        p = {"compress_w": xavier(self.d_model, cd, (self.d_model, cd)),
             "compress_b": np.zeros(cd)}
        for i, n_in in ((1, cd), (2, hid)):
            s = 1.0 / np.sqrt(hid)
            p[f"lstm{i}_wx"] = rng.uniform(-s, s, (n_in, 4 * hid))
            p[f"lstm{i}_wh"] = rng.uniform(-s, s, (hid, 4 * hid))
            b = np.zeros(4 * hid)
            b[hid : 2 * hid] = 1.0
            p[f"lstm{i}_b"] = b
        for name in ("attn_wq", "attn_wk", "attn_wv"):
            p[name] = xavier(hid, hid, (hid, hid))
        p["head_w"] = xavier(hid, self.num_experts,
                             (self.num_moe_layers, hid, self.num_experts))
        p["head_b"] = np.zeros((self.num_moe_layers, self.num_experts))
        return p

    def param_bytes(self) -> int:
        return sum(v.size for v in self.params.values()) * 8

    def packed(self, device) -> torch.Tensor:
        key = str(device)
        if key not in self._packed:
            flat = np.concatenate([np.ascontiguousarray(self.params[n], dtype=np.float64).ravel()
                                   for n in PARAM_ORDER])
            c = self.config
            want = _lib.load().sida_hash_param_count(self.d_model, c.compress_dim, c.lstm_hidden,
                                                     self.num_moe_layers, self.num_experts)
            if flat.size != want:
                raise ContractError(f"predictor params hold {flat.size} values, expected {want}")
            self._packed[key] = torch.from_numpy(flat).to(device)
        return self._packed[key]

    def tables(self, model, device, stream):
        """Per-model folding tables of sida_hash_prepare (cached): the compress
        FC and layer-1 input projection folded into vocabulary / position rows
        of ``model``'s bf16 embedding tables (``model`` None: the caller-
        embedding path, which only needs the bias row and packed [Wq|Wk|Wv]).
        Returns (tables, vocab, max_len)."""
        key = (str(device), id(model))
        hit = self._tables.get(key) if hasattr(self, "_tables") else None
        if hit is not None and hit[0] is model:
            return hit[1], hit[2], hit[3]
        if not hasattr(self, "_tables"):
            self._tables = {}
        h = _lib.lib()
        c = self.config
        vocab = model.config.vocab_size if model is not None else 0
        tmax = model.config.max_seq_len if model is not None else 0
        if model is not None and model.config.d_model != self.d_model:
            raise ContractError("predictor d_model does not match the model")
        n = h.sida_hash_tables_count(vocab, tmax, c.lstm_hidden, self.num_moe_layers,
                                     self.num_experts)
        tab = torch.empty(n, dtype=torch.float64, device=device)
        with torch.cuda.stream(stream):
            _lib.check(h.sida_hash_prepare(
                self.packed(device).data_ptr(), _lib.ptr(model.tok_emb) if model else None,
                _lib.ptr(model.pos_emb) if model else None, vocab, tmax, self.d_model,
                c.compress_dim, c.lstm_hidden, self.num_moe_layers, self.num_experts,
                tab.data_ptr(), stream.cuda_stream))
        self._tables[key] = (model, tab, vocab, tmax)
        return tab, vocab, tmax


def _fresh(device):
    """Allocator of per-table buffers from the caching allocator."""
    def new(name, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=device)
    return new


class TableSlot:
    """Long-lived device buffers one hash table is built in (one slot of a
    `DeviceTableRing`); grows to the largest batch seen. ``consumed`` is the
    event after which the slot's previous table is no longer read."""

    def __init__(self, device):
        self.device = device
        self.bufs: dict = {}
        self.consumed = None
        self.busy = False
        self.table = None  # weakref to the table built in the slot
        # sticky permute contract flag of every table built in this slot
        self.err = torch.zeros(1, dtype=torch.int32, device=device)

    def get(self, name, shape, dtype):
        n = int(np.prod(shape))
        buf = self.bufs.get(name)
        if buf is None or buf.numel() < n or buf.dtype != dtype:
            buf = torch.empty(max(n, 1), dtype=dtype, device=self.device)
            self.bufs[name] = buf
        return buf[:n].view(shape)

    def upload_tokens(self, toks: np.ndarray, stream) -> torch.Tensor:
        """Host token ids -> this slot's device token buffer through the slot's
        own pinned staging buffer (no pinned allocation per batch; the host
        rewrites it only after the previous copy out of it has completed)."""
        n = toks.size
        st = getattr(self, "_stage", None)
        if st is None or st.numel() < n:
            st = torch.empty(max(n, 1), dtype=torch.int32, pin_memory=True)
            self._stage, self._stage_ev = st, None
        if self._stage_ev is not None:
            self._stage_ev.synchronize()
        st[:n].numpy()[:] = toks
        dev = self.get("tokens", (n,), torch.int32)
        with torch.cuda.stream(stream):
            # SM copy from pinned memory: no copy-engine queueing behind expert copies
            _lib.check(_lib.lib().sida_copy_sm(dev.data_ptr(), st.data_ptr(), 4 * n,
                                               stream.cuda_stream))
            self._stage_ev = torch.cuda.Event()
            self._stage_ev.record(stream)
        return dev


class DeviceTableRing:
    """The device-resident form of the hash-table queue (ref pipeline.py:53-84
    holds host tables in a bounded FIFO): ``capacity`` table slots of device
    buffers (`TableSlot`), written by the hash stream and read by the compute
    stream. Back-pressure is device-side: before a slot is rewritten the hash
    stream waits on the event recorded after the forward that read its
    previous table (`release`, done by the engines' forward), so no host
    thread, lock or queue object sits between hashing and inference. Tables
    are produced in strictly increasing batch_id order and a slot whose table
    was not consumed yet is never overwritten (ContractError), like
    HashTableQueue.put / get."""

    def __init__(self, capacity: int, device, strict: bool = True):
        if capacity < 1:
            raise ContractError("queue capacity must be >= 1")
        self.capacity = capacity
        self.slots = [TableSlot(device) for _ in range(capacity)]
        self.n = 0
        self._last_id: int | None = None
        # strict: the queue contract (ordered ids, never overwrite an unread
        # table). Non-strict (an engine's own ring): a full ring or an
        # out-of-order id builds the table in fresh allocations instead.
        self.strict = strict

    def restart(self) -> None:
        """Start a new stream of batch ids (a new serve_sida call on a ring kept
        warm across calls). Tables a previous call left unconsumed (it raised)
        are abandoned once the device is idle."""
        if any(s.busy for s in self.slots):
            torch.cuda.synchronize(self.slots[0].device)
            for s in self.slots:
                s.busy = False
        self._last_id = None

    def produce(self, predictor, model, lengths, eval_top_k: int, stream, batch_id: int,
                tokens_dev=None, batch=None, host_ids: bool = False):
        """Hash + permute one batch into the next slot on ``stream``: device
        tokens (``tokens_dev``) or a host ``batch`` (tokens uploaded into the
        slot). ``host_ids`` also starts an async copy of ids / alphas to pinned
        memory (read after the slot is reused, e.g. for the hit rate)."""
        if eval_top_k < 1 or eval_top_k > predictor.num_experts:
            raise ContractError(f"k={eval_top_k} out of range for width-{predictor.num_experts} rows")
        slot = self.slots[self.n % self.capacity]
        in_order = self._last_id is None or batch_id > self._last_id
        if not self.strict and (slot.busy or not in_order):
            with torch.cuda.stream(stream):
                if tokens_dev is None:
                    toks = model.validate_tokens(batch)
                    tokens_dev = torch.from_numpy(toks).pin_memory().to(model.device,
                                                                        non_blocking=True)
                return hash_device(predictor, model, tokens_dev, list(lengths), eval_top_k,
                                   batch_id, stream)
        if not in_order:
            raise ContractError("hash tables must be enqueued in batch_id order")
        if slot.busy:
            raise ContractError("hash-table ring full: forward the oldest table first")
        self._last_id = batch_id
        self.n += 1
        with torch.cuda.stream(stream):
            if slot.consumed is not None:
                stream.wait_event(slot.consumed)
            if tokens_dev is None:
                tokens_dev = slot.upload_tokens(model.validate_tokens(batch), stream)
            table = hash_device(predictor, model, tokens_dev, list(lengths), eval_top_k,
                                batch_id, stream, slot=slot)
            if host_ids:
                dt = table._dev
                ids = torch.empty(dt.ids.shape, dtype=dt.ids.dtype, pin_memory=True)
                al = torch.empty(dt.alpha.shape, dtype=dt.alpha.dtype, pin_memory=True)
                ids.copy_(dt.ids, non_blocking=True)
                al.copy_(dt.alpha, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                table._host_async = (ids, al, ev)
        prev = slot.table() if slot.table is not None else None
        if prev is not None:
            prev._stale = True  # its device arrays now hold this batch
        slot.busy = True
        slot.table = weakref.ref(table)
        table._slot = slot
        return table

    @staticmethod
    def release(table, stream) -> None:
        """Mark the table's slot reusable once ``stream`` (the consumer) has
        passed this point (no-op for tables outside a ring)."""
        slot = getattr(table, "_slot", None)
        if slot is None:
            return
        ev = torch.cuda.Event()
        ev.record(stream)
        slot.consumed = ev
        slot.busy = False

    def error_flags(self):
        return [s.err for s in self.slots]


class DeviceTable:
    """Device half of an ExpertHashTable: ids/alphas plus the per-layer
    permutation (hist, off, perm, inv, alpha_perm) and the event after which
    all of it is valid on any stream."""

    def __init__(self, ids, alpha, alpha_f32, n_tokens, k, tokens=None):
        self.ids = ids              # int32 (L, N, k)
        self.alpha = alpha          # float64 (L, N, k)
        self.alpha_f32 = alpha_f32  # float32 (L, N, k)
        self.num_layers = ids.shape[0]
        self.n_tokens = n_tokens
        self.k = k
        self.tokens = tokens        # int32 device tokens when built by the GPU hasher
        self.hist = self.off = self.perm = self.inv = self.alpha_perm = None
        self.err = None             # int32 (1,): set by the permute on an out-of-range id
        self.ready = torch.cuda.Event()

    def permute(self, num_experts: int, stream, slot: "TableSlot | None" = None) -> None:
        h = _lib.lib()
        L, rows = self.num_layers, self.n_tokens * self.k
        dev = self.ids.device
        new = slot.get if slot is not None else _fresh(dev)
        self.hist = new("hist", (L, num_experts), torch.int32)
        self.off = new("off", (L, num_experts + 1), torch.int32)
        self.perm = new("perm", (L, rows), torch.int32)
        self.inv = new("inv", (L, rows), torch.int32)
        self.alpha_perm = new("alpha_perm", (L, rows), torch.float32)
        ws_bytes = h.sida_permute_workspace_bytes(L, rows, num_experts)
        ws = new("perm_ws", (ws_bytes,), torch.uint8)
        # sticky contract flag (never cleared by the kernel): the slot's own,
        # or a fresh zeroed one per table
        self.err = slot.err if slot is not None else torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(h.sida_permute_hist(
            self.ids.data_ptr(), L, rows, num_experts, self.alpha_f32.data_ptr(),
            self.hist.data_ptr(), self.off.data_ptr(), self.perm.data_ptr(), self.inv.data_ptr(),
            self.alpha_perm.data_ptr(), self.err.data_ptr(), ws.data_ptr(), ws_bytes,
            stream.cuda_stream))
        ws.record_stream(stream)
        self.ready.record(stream)

    def use_on(self, stream) -> None:
        """Mark the table's buffers as in use on ``stream`` (caching-allocator
        safety when the table was built on another stream)."""
        for t in (self.ids, self.alpha, self.alpha_f32, self.hist, self.off, self.perm, self.inv,
                  self.alpha_perm, self.tokens, self.err):
            if t is not None:
                t.record_stream(stream)

    def layer(self, layer: int):
        return self.off[layer], self.perm[layer], self.alpha_perm[layer]

    def hist_host(self) -> np.ndarray:
        """(L, K) expert histograms on the host: one D2H per table (waits for
        the permute), cached -- the planner and the per-layer paths read it."""
        if getattr(self, "_hist_host", None) is None:
            self.ready.synchronize()
            self._hist_host = self.hist.cpu().numpy()
        return self._hist_host

    def tokens_for(self, model: MoEModel, batch: SequenceBatch, stream=None) -> torch.Tensor:
        """The batch's int32 tokens on the device. A table built on the host
        has none: they are copied on ``stream`` (the stream that will read
        them; default the current one), so no other stream can race the copy."""
        if self.tokens is None:
            toks = model.validate_tokens(batch)
            st = stream or torch.cuda.current_stream(model.device)
            with torch.cuda.stream(st):
                self.tokens = torch.from_numpy(toks).pin_memory().to(model.device,
                                                                     non_blocking=True)
        return self.tokens


class ExpertHashTable:
    """Predicted (expert id, alpha) per (layer, token) for one batch
    (ref predictor.py:61-126). Constructed either from numpy arrays (the
    reference's form) or by the GPU hasher, in which case the arrays live on
    the device and the numpy views are fetched on first access."""

    def __init__(self, batch_id: int, lengths: list[int], ids=None, alphas=None, *,
                 device_table: DeviceTable | None = None):
        self.batch_id = int(batch_id)
        self.lengths = [int(n) for n in lengths]
        self._ids = None if ids is None else np.asarray(ids, dtype=np.int64)
        self._alphas = None if alphas is None else np.asarray(alphas, dtype=np.float64)
        self._dev = device_table
        self._hist = None
        if self._ids is None and self._dev is None:
            raise ContractError("hash table needs ids or a device table")

    # -- numpy view (boundary iv) ----------------------------------------------------
    def _check_live(self) -> None:
        if getattr(self, "_stale", False):
            raise ContractError(f"hash table {self.batch_id}: its device-ring slot was reused; "
                                "read ids/alphas before the ring wraps (or build it outside a ring)")

    def _from_async(self) -> bool:
        pend = getattr(self, "_host_async", None)
        if pend is None:
            return False
        ids, al, ev = pend
        ev.synchronize()
        self._ids = ids.numpy().astype(np.int64)
        self._alphas = al.numpy().copy()
        self._host_async = None
        return True

    @property
    def ids(self) -> np.ndarray:
        if self._ids is None and not self._from_async():
            self._check_live()
            self._dev.ready.synchronize()
            self._ids = self._dev.ids.cpu().numpy().astype(np.int64)
        return self._ids

    @property
    def alphas(self) -> np.ndarray:
        if self._alphas is None and not self._from_async():
            self._check_live()
            self._dev.ready.synchronize()
            self._alphas = self._dev.alpha.cpu().numpy()
        return self._alphas

    @property
    def num_layers(self) -> int:
        return self._dev.num_layers if self._dev is not None else self._ids.shape[0]

    @property
    def eval_top_k(self) -> int:
        return self._dev.k if self._dev is not None else self._ids.shape[2]

    @property
    def num_tokens(self) -> int:
        return self._dev.n_tokens if self._dev is not None else self._ids.shape[1]

    def sequence_slice(self, offset: int, t_len: int):
        if offset + t_len > self.num_tokens:
            raise ContractError("hash table does not cover the requested tokens")
        return self.ids[:, offset : offset + t_len], self.alphas[:, offset : offset + t_len]

    def histogram(self) -> np.ndarray:
        """(L, K) per-layer expert counts (device hist when available)."""
        if self._hist is None:
            if self._dev is not None and self._dev.hist is not None:
                self._hist = self._dev.hist_host()
            else:
                K = int(self.ids.max()) + 1
                self._hist = np.stack([np.bincount(self.ids[l].ravel(), minlength=K)
                                       for l in range(self.num_layers)])
        return self._hist

    def required_experts(self) -> set[tuple[int, int]]:
        """ref predictor.py:89-94."""
        return {(l, int(e)) for l, row in enumerate(self.histogram()) for e in np.nonzero(row)[0]}

    def required_by_layer(self) -> list[set[int]]:
        """ref predictor.py:96-100 (sorted sets of the experts each layer needs)."""
        return [{int(e) for e in np.nonzero(row)[0]} for row in self.histogram()]

    def to_json(self) -> str:
        """ref predictor.py:102-112."""
        entries = []
        ids, al = self.ids, self.alphas
        for layer in range(ids.shape[0]):
            for tok in range(ids.shape[1]):
                entries.append([layer, tok, [[int(e), float(a)]
                                             for e, a in zip(ids[layer, tok], al[layer, tok])]])
        return json.dumps({"batch_id": self.batch_id, "lengths": self.lengths, "entries": entries})

    @classmethod
    def from_json(cls, text: str) -> "ExpertHashTable":
        """ref predictor.py:114-126."""
        obj = json.loads(text)
        lengths = [int(x) for x in obj["lengths"]]
        layers = 1 + max(e[0] for e in obj["entries"])
        k = len(obj["entries"][0][2])
        ids = np.zeros((layers, sum(lengths), k), dtype=np.int64)
        alphas = np.zeros((layers, sum(lengths), k))
        for layer, tok, pairs in obj["entries"]:
            ids[layer, tok] = [p[0] for p in pairs]
            alphas[layer, tok] = [p[1] for p in pairs]
        return cls(int(obj["batch_id"]), lengths, ids, alphas)

    # -- device view -----------------------------------------------------------------
    def on_device(self, model: MoEModel, stream=None) -> DeviceTable:
        """The device table (uploading + permuting a host-built table once)."""
        if self._dev is None:
            st = stream or torch.cuda.current_stream(model.device)
            ids = self._ids
            K = model.config.num_experts
            if ids.size and (ids.min() < 0 or ids.max() >= K):
                raise ContractError("expert index out of range")
            if self._alphas is None or np.any(self._alphas < 0):
                raise ContractError("scaling factors must be non-negative")
            with torch.cuda.stream(st):
                d_ids = torch.from_numpy(ids.astype(np.int32)).to(model.device)
                d_al = torch.from_numpy(self._alphas).to(model.device)
                dt = DeviceTable(d_ids, d_al, d_al.float(), ids.shape[1], ids.shape[2])
                dt.permute(K, st)
            self._dev = dt
        return self._dev


def build_hash_table(predictor: PredictorNet, batch: SequenceBatch, eval_top_k: int, embed_fn,
                     stream=None) -> ExpertHashTable:
    """Top-k expert ids and alphas per (layer, token) (ref predictor.py:373-399).

    ``embed_fn`` is normally ``model.embed`` of a GPU `MoEModel`: the kernel
    then reads the model's bf16 embedding tables directly. Any other callable
    is evaluated on the host per sequence and its float64 embeddings are
    uploaded. Alphas are the raw softmax probabilities at the ids."""
    if eval_top_k < 1:
        raise ContractError("eval_top_k must be >= 1")
    if eval_top_k > predictor.num_experts:
        raise ContractError(f"k={eval_top_k} out of range for width-{predictor.num_experts} rows")
    model = getattr(embed_fn, "__self__", None)
    use_tables = isinstance(model, MoEModel) and getattr(embed_fn, "__name__", "") == "embed"
    device = model.device if use_tables else torch.device("cuda", torch.cuda.current_device())
    st = stream or torch.cuda.current_stream(device)
    lengths = batch.lengths
    if not lengths or min(lengths) < 1:
        raise ContractError("empty sequence")
    n_tok = sum(lengths)
    with torch.cuda.stream(st):
        tokens = None
        emb = None
        if use_tables:
            toks = model.validate_tokens(batch)
            tokens = torch.from_numpy(toks).pin_memory().to(device, non_blocking=True)
        else:
            host = np.concatenate([np.asarray(embed_fn(s), dtype=np.float64) for s in batch.sequences])
            if host.shape != (n_tok, predictor.d_model) or not np.all(np.isfinite(host)):
                raise ContractError("predictor input must be finite (T, d_model) embeddings")
            emb = torch.from_numpy(host).to(device)
    return hash_device(predictor, model if use_tables else None, tokens, lengths, eval_top_k,
                       batch.batch_id, st, emb=emb, device=device)


def hash_device(predictor: PredictorNet, model: MoEModel | None, tokens, lengths, eval_top_k: int,
                batch_id: int, stream, emb=None, device=None,
                slot: TableSlot | None = None) -> ExpertHashTable:
    """Hash + permute for tokens already resident in HBM (int32 ``tokens`` on
    the device, or float64 embeddings ``emb``), enqueued on ``stream``;
    ``slot`` (a `DeviceTableRing` slot) holds the outputs instead of fresh
    allocations."""
    h = _lib.lib()
    st = stream
    device = device or (model.device if model is not None else emb.device)
    n_tok, n_seq, max_len = sum(lengths), len(lengths), max(lengths)
    c = predictor.config
    L, K = predictor.num_moe_layers, predictor.num_experts
    off = np.zeros(n_seq + 1, dtype=np.int32)
    np.cumsum(lengths, out=off[1:])
    use_tables = model is not None
    with torch.cuda.stream(st):
        new = slot.get if slot is not None else _fresh(device)
        # as a kernel-parameter write, not an H2D memcpy: it must not queue
        # behind expert copies on the copy engines (sida_poke_i32)
        seq_off = new("seq_off", (n_seq + 1,), torch.int32)
        _lib.check(h.sida_poke_i32(seq_off.data_ptr(), off.ctypes.data, n_seq + 1, st.cuda_stream))
        ids = new("ids", (L, n_tok, eval_top_k), torch.int32)
        alpha = new("alpha", (L, n_tok, eval_top_k), torch.float64)
        alpha_f32 = new("alpha_f32", (L, n_tok, eval_top_k), torch.float32)
        ws_bytes = h.sida_hash_workspace_bytes(n_tok, n_seq, max_len, predictor.d_model,
                                               c.compress_dim, c.lstm_hidden, L, K)
        ws = new("hash_ws", (ws_bytes,), torch.uint8)
        params = predictor.packed(device)
        tables, vocab, tmax = predictor.tables(model, device, st)
        _lib.check(h.sida_hash_forward(
            params.data_ptr(), tables.data_ptr(), vocab, tmax, _lib.ptr(emb), _lib.ptr(tokens),
            seq_off.data_ptr(), n_seq, n_tok, max_len, predictor.d_model, c.compress_dim,
            c.lstm_hidden, L, K, eval_top_k, ids.data_ptr(), alpha.data_ptr(),
            alpha_f32.data_ptr(), ws.data_ptr(), ws_bytes, st.cuda_stream))
        dt = DeviceTable(ids, alpha, alpha_f32, n_tok, eval_top_k, tokens=tokens)
        dt.permute(K, st, slot=slot)
        ws.record_stream(st)
    return ExpertHashTable(batch_id, lengths, device_table=dt)


class PredictorHasher:
    """Binds a predictor to an embedding source (ref predictor.py:402-410)."""

    def __init__(self, predictor: PredictorNet, embed_fn, stream=None):
        self.predictor = predictor
        self.embed_fn = embed_fn
        self.stream = stream

    def build_table(self, batch: SequenceBatch, eval_top_k: int) -> ExpertHashTable:
        return build_hash_table(self.predictor, batch, eval_top_k, self.embed_fn, self.stream)


class OracleHasher:
    """The teacher routers as the hash function (ref predictor.py:413-426):
    a router-mode forward on the GPU whose per-layer top-``eval_top_k``
    selections (descending probability, ties to the lower index) and
    probabilities become the table. Upper-bounds hit rate and fidelity."""

    def __init__(self, model: MoEModel, stream=None, store=None):
        self.model = model
        self.stream = stream
        self.store = store

    def build_table(self, batch: SequenceBatch, eval_top_k: int) -> ExpertHashTable:
        c = self.model.config
        if not 1 <= eval_top_k <= c.num_experts:
            raise ContractError(f"k={eval_top_k} out of range for width-{c.num_experts} rows")
        st = self.stream or torch.cuda.current_stream(self.model.device)
        with torch.cuda.stream(st):
            lay = BatchLayout.from_batch(self.model, batch)
            ktop = max(eval_top_k, c.routing_k)
            _, ids, al, _ = router_forward(self.model, lay, ktop, store=self.store, stream=st)
            ids = ids[:, :, :eval_top_k].contiguous()
            al = al[:, :, :eval_top_k].contiguous()
            dt = DeviceTable(ids, al, al.float(), lay.n_tokens, eval_top_k, tokens=lay.tokens)
            dt.permute(c.num_experts, st)
        return ExpertHashTable(batch.batch_id, batch.lengths, device_table=dt)


def hash_hit_rate(tables: list, traces: list, k: int) -> float:
    """Fraction of (layer, token) whose teacher top-1 expert is among the
    first k predicted ids (ref predictor.py:429-449)."""
    if len(tables) != len(traces):
        raise CoverageError("table/trace counts differ")
    if k < 1:
        raise ContractError("k must be >= 1")
    hits = total = 0
    for table, trace in zip(tables, traces):
        if table.lengths != list(trace.lengths):
            raise CoverageError("table and trace cover different sequences")
        if table.num_layers != trace.num_layers:
            raise CoverageError("table and trace cover different layer counts")
        if k > table.eval_top_k:
            raise CoverageError(f"k={k} exceeds table width {table.eval_top_k}")
        top1 = trace.selected[:, :, 0]
        hits += int(np.sum(np.any(table.ids[:, :, :k] == top1[:, :, None], axis=-1)))
        total += top1.size
    if total == 0:
        raise CoverageError("empty coverage")
    return hits / total
