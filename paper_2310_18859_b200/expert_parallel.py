"""Expert parallelism across the GPUs of one box.

Rank r owns experts [r*K/G, (r+1)*K/G) of every MoE layer (contiguous blocks),
holds only those in its HBM slot arena, and serves its own batch stream
(hash, embed and attention are local). Per batch the ranks exchange their
(L, K) expert histograms once -- SiDA knows every layer's routing before
inference starts, so no per-layer size handshake is needed. Per layer:

  x_perm  = gather(x_attn)            rows already grouped by expert, hence by
                                      destination rank (experts are contiguous)
  recv    = all_to_all(x_perm)        bf16 rows, splits from the histograms
  x_local = regroup(recv)             (source, expert) order -> expert-major
  y_recv  = grouped FFN (local experts); the GEMM2 epilogue writes each row
            straight back to its receive position (row_map) as bf16
  y_back  = all_to_all(y_recv)        back to the source rank, x_perm order
  out     = x_attn + sum_r alpha * y  sida_unpermute_combine (ranks in order)

The transport is NCCL over NVLink (`NcclTransport`, device tensors) in
production; `GlooTransport` stages through host memory so the same data path
runs (and is tested) with several ranks on one GPU or on CPU-only hosts.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .errors import ContractError, UnservableError
from .moe import BatchLayout, MoEModel
from .offload import ExpertStore, MemoryBudget, ResidencyState, apply_group_inplace, plan_placement


# ----------------------------------------------------------------------- host math
def owner_block(num_experts: int, world: int) -> int:
    if num_experts % world:
        raise ContractError(f"{num_experts} experts do not split evenly over {world} ranks")
    return num_experts // world


def ep_splits(counts: np.ndarray, layer: int, rank: int, world: int):
    """Row counts this rank sends to / receives from every rank for ``layer``.

    ``counts`` is (G, L, K): every rank's per-layer expert histogram of its own
    (token, rank) rows."""
    kl = owner_block(counts.shape[2], world)
    own = counts[rank, layer].reshape(world, kl).sum(axis=1)          # to each owner
    recv = counts[:, layer, rank * kl:(rank + 1) * kl].sum(axis=1)    # from each source
    return own.astype(np.int64), recv.astype(np.int64)


def ep_regroup(counts: np.ndarray, layer: int, rank: int, world: int):
    """Receive buffer (source-major, then local expert) -> expert-major order.

    Returns (src (R,) int32: receive position of each expert-major row,
    off (Kl+1,) int32 expert offsets of the expert-major rows)."""
    kl = owner_block(counts.shape[2], world)
    c = counts[:, layer, rank * kl:(rank + 1) * kl].astype(np.int64)  # (G, Kl)
    recv_off = np.zeros((world, kl), dtype=np.int64)                  # start of (g, e) in recv
    flat = c.reshape(-1)
    starts = np.concatenate([[0], np.cumsum(flat)[:-1]]).reshape(world, kl)
    recv_off[:] = starts
    per_e = c.sum(axis=0)
    off = np.zeros(kl + 1, dtype=np.int32)
    np.cumsum(per_e, out=off[1:])
    src = np.empty(int(per_e.sum()), dtype=np.int32)
    for e in range(kl):
        pos = off[e]
        for g in range(world):
            n = int(c[g, e])
            src[pos:pos + n] = np.arange(recv_off[g, e], recv_off[g, e] + n, dtype=np.int32)
            pos += n
    return src, off


# ----------------------------------------------------------------------- transports
class NcclTransport:
    """Device tensors through torch.distributed (backend nccl)."""

    def __init__(self, group=None):
        self.group = group

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        world = dist.get_world_size(self.group)
        out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        return out

    def all_to_all(self, send: torch.Tensor, send_rows, recv_rows) -> torch.Tensor:
        recv = torch.empty((int(sum(recv_rows)),) + tuple(send.shape[1:]), dtype=send.dtype,
                           device=send.device)
        dist.all_to_all_single(recv, send, output_split_sizes=[int(v) for v in recv_rows],
                               input_split_sizes=[int(v) for v in send_rows], group=self.group)
        return recv


class GlooTransport(NcclTransport):
    """Same interface, staged through host memory (gloo collectives)."""

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        h = t.detach().cpu().contiguous()
        world = dist.get_world_size(self.group)
        parts = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(parts, h, group=self.group)
        return torch.stack(parts).to(t.device)

    def all_to_all(self, send: torch.Tensor, send_rows, recv_rows) -> torch.Tensor:
        hs = send.detach().cpu().contiguous()
        raw = hs.view(torch.uint8).reshape(hs.shape[0], -1)  # gloo moves raw bytes per row
        recv = torch.empty((int(sum(recv_rows)), raw.shape[1]), dtype=torch.uint8)
        dist.all_to_all_single(recv, raw, output_split_sizes=[int(v) for v in recv_rows],
                               input_split_sizes=[int(v) for v in send_rows], group=self.group)
        out = recv.view(send.dtype).reshape((-1,) + tuple(send.shape[1:]))
        return out.to(send.device)


class PeerTransport(NcclTransport):
    """No collective on the data path. Every rank maps
    every other rank's expert-major receive buffers (two, by layer parity),
    its return buffer and its flag words through CUDA IPC (NVLink peer
    mappings on a multi-GPU box); the attention output projection writes each
    token's expert input straight into the owner's receive buffer and the
    owner's GEMM2 epilogue writes each expert output straight back into the
    source's return buffer. Stream-ordered release/acquire flags
    (sida_peer_signal / sida_peer_wait) separate producer and consumer. Only
    the per-batch (L, K) histograms use torch.distributed (``control``)."""

    peer = True

    def __init__(self, control=None, group=None):
        super().__init__(group)
        self.control = control or NcclTransport(group)
        self.ready = False
        self._opened: list = []

    def all_gather(self, t):
        return self.control.all_gather(t)

    def setup(self, model: MoEModel, rows_per_rank: int) -> None:
        """Allocate and cross-map the buffers for up to ``rows_per_rank``
        (token, rank) rows per source rank and batch."""
        import ctypes as C

        h = _lib.lib()
        world, me = dist.get_world_size(self.group), dist.get_rank(self.group)
        d, dev = model.config.d_model, model.device
        self.world, self.me = world, me
        self.cap_y = int(rows_per_rank)
        self.cap_x = world * self.cap_y
        self.xloc = [torch.empty((self.cap_x, d), dtype=torch.bfloat16, device=dev)
                     for _ in range(2)]
        self.yback = torch.empty((self.cap_y, d), dtype=torch.bfloat16, device=dev)
        self.flags = torch.zeros(world, dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)
        nb = int(h.sida_ipc_handle_bytes())

        def handle(t):
            buf = C.create_string_buffer(nb)
            off = C.c_size_t(0)
            _lib.check(h.sida_ipc_handle(C.c_void_p(t.data_ptr()), buf, C.byref(off)))
            return buf.raw, off.value

        mine = [handle(t) for t in (self.xloc[0], self.xloc[1], self.yback, self.flags)]
        allh: list = [None] * world
        dist.all_gather_object(allh, mine, group=self.group)
        ptrs = []
        for q in range(world):
            row = []
            for i, t in enumerate((self.xloc[0], self.xloc[1], self.yback, self.flags)):
                if q == me:
                    row.append(t.data_ptr())
                    continue
                base, ptr = C.c_void_p(), C.c_void_p()
                raw, off = allh[q][i]
                _lib.check(h.sida_ipc_open(raw, off, C.byref(base), C.byref(ptr)))
                self._opened.append(base.value)
                row.append(ptr.value)
            ptrs.append(row)
        as_dev = lambda col: torch.tensor([ptrs[q][col] for q in range(world)],  # noqa: E731
                                          dtype=torch.int64, device=dev)
        self.xloc_peers = [as_dev(0), as_dev(1)]
        self.yback_peers = as_dev(2)
        self.flag_peers = as_dev(3)
        self.epoch = 0
        self.ready = True
        dist.barrier(group=self.group)

    def exchange_done(self, stream) -> None:
        """Publish this rank's stores of the current exchange and wait for
        every rank's (both stream-ordered, no host synchronisation)."""
        h = _lib.lib()
        self.epoch += 1
        _lib.check(h.sida_peer_signal(self.flag_peers.data_ptr(), self.world, self.me, self.epoch,
                                      stream.cuda_stream))
        _lib.check(h.sida_peer_wait(self.flags.data_ptr(), self.world, self.epoch,
                                    stream.cuda_stream))


def ep_peer_maps(counts: np.ndarray, layer: int, rank: int, world: int, stride_x: int,
                 stride_y: int):
    """Host half of the peer exchange maps for one layer, from the (G, L, K)
    histograms every rank holds after the per-batch all-gather:

    dispatch: my expert-sorted row p of (global) expert e goes to owner
      q = e // kl at row  loc_off_q[e - q kl] + sum_{g < me} c[g, e]  of its
      receive buffer (expert-major, source-minor: ep_regroup's layout) ->
      segments (start off_me[e], value q * stride_x + that row);
    return: my received row in block (local expert el, source g) goes back to
      g's expert-sorted position off_g[e] -> segments (block start, value
      g * stride_y + off_g[e]);
    plus this rank's local expert offsets (kl + 1) and received row count."""
    kl = owner_block(counts.shape[2], world)
    c = counts[:, layer, :].astype(np.int64)                        # (G, K)
    K = c.shape[1]
    off_src = np.zeros((world, K + 1), dtype=np.int64)              # each source's expert-sorted offsets
    np.cumsum(c, axis=1, out=off_src[:, 1:])
    tot = c.sum(axis=0)                                             # rows per expert, all sources
    before = np.cumsum(c, axis=0) - c                               # sum_{g' < g} c[g', e]
    d_start = off_src[rank].astype(np.int32)                        # (K + 1)
    d_val = np.empty(K, dtype=np.int64)
    for q in range(world):
        blk = tot[q * kl:(q + 1) * kl]
        loc = np.concatenate([[0], np.cumsum(blk)[:-1]])
        d_val[q * kl:(q + 1) * kl] = q * stride_x + loc + before[rank, q * kl:(q + 1) * kl]
    lo = rank * kl
    off_l = np.zeros(kl + 1, dtype=np.int32)
    np.cumsum(tot[lo:lo + kl], out=off_l[1:])
    r_start = np.empty(kl * world + 1, dtype=np.int32)
    r_val = np.empty(kl * world, dtype=np.int64)
    for el in range(kl):
        e = lo + el
        for g in range(world):
            b = el * world + g
            r_start[b] = off_l[el] + before[g, e]
            r_val[b] = g * stride_y + off_src[g, e]
    r_start[-1] = off_l[-1]
    return (d_start, d_val.astype(np.int32), r_start, r_val.astype(np.int32), off_l,
            int(off_l[-1]))


# ----------------------------------------------------------------------- engine
class _LocalTable:
    """`required_by_layer` view restricted to this rank's experts (global ids)."""

    def __init__(self, counts: np.ndarray, rank: int, kl: int):
        tot = counts.sum(axis=0)  # (L, K)
        lo = rank * kl
        self._req = [{lo + e for e in np.nonzero(tot[l, lo:lo + kl])[0]} for l in range(tot.shape[0])]

    def required_by_layer(self):
        return self._req

    def required_experts(self):
        return {(l, e) for l, s in enumerate(self._req) for e in s}


class _GroupIssuer:
    """Slot bookkeeping of one batch's plan, one group at a time, in plan
    order (like SidaEngine._issue): group l is applied when layer l starts
    (and group l+1 right after it when prefetchable, ref pipeline.py:246-253),
    so an expert a later group evicts is still in its slot when its own layer
    reads the slot row. Each load waits on its slot's last reader."""

    def __init__(self, eng: "ExpertParallelEngine", plan, required):
        self.eng, self.plan, self.required = eng, plan, required
        self.issued = [False] * len(plan.groups)
        self.done: list = [None] * len(plan.groups)

    def _issue(self, idx: int) -> None:
        eng = self.eng
        g = self.plan.groups[idx]
        eb = eng.model.expert_bytes_each()
        apply_group_inplace(eng.state, g, eng.budget.fast_tier_bytes, eb)
        eng.peak = max(eng.peak, eng.state.used_bytes)
        loads = []
        for op, key in g.steps:
            if op == "evict":
                eng.store.free_slot(key)
            else:
                loads.append((key, eng.store.take_slot(key)))
        self.done[idx] = eng.store.enqueue_loads(loads)
        self.issued[idx] = True

    def issue_for(self, layer: int):
        """Issue this layer's group (and the next one when prefetchable);
        returns the done event of this layer's copies (or None)."""
        if not self.issued[layer]:
            self._issue(layer)
        nxt = layer + 1
        if nxt < len(self.plan.groups) and self.plan.groups[nxt].prefetchable and not self.issued[nxt]:
            self._issue(nxt)
        return self.done[layer]

    def slot_row(self, layer: int) -> np.ndarray:
        """Local expert -> slot of ``layer``, taken right before its FFN;
        every expert the layer routes rows to must be resident."""
        eng = self.eng
        lo = eng.rank * eng.kl
        row = np.full(eng.kl, -1, dtype=np.int32)
        for e in self.required[layer]:
            slot = eng.store.slot_of.get((layer, e))
            if slot is None:
                raise ContractError(f"plan/state mismatch: expert {(layer, e)} not resident")
            row[e - lo] = slot
        return row


class ExpertParallelEngine:
    """SiDA serving with experts sharded over the ranks of ``group``.

    Residency is per rank over its own expert block (the reference planner on
    the union of every rank's needs for those experts). A layer whose local
    working set exceeds the budget is rejected (waves are single-GPU only)."""

    def __init__(self, model: MoEModel, predictor, budget: MemoryBudget, transport=None,
                 group=None, eval_top_k: int = 1):
        from .engine import SidaEngine  # streams + hash plumbing

        self.model = model
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.kl = owner_block(model.config.num_experts, self.world)
        self.transport = transport or NcclTransport(group)
        self.base = SidaEngine(model, predictor, budget, eval_top_k)
        self.store: ExpertStore = self.base.store
        self.state = ResidencyState()
        self.budget = budget
        self.peak = 0

    def hash_tokens(self, batch_id, tokens_dev, lengths):
        return self.base.hash_tokens(batch_id, tokens_dev, lengths)

    def forward(self, table, lengths, tokens_dev=None, batch=None):
        model, store, budget = self.model, self.store, self.budget
        c = model.config
        h = _lib.lib()
        eb = model.expert_bytes_each()
        cs = self.base.compute_stream
        dt = table.on_device(model, stream=self.base.hash_stream)
        if tokens_dev is None:
            tokens_dev = dt.tokens_for(model, batch, cs)
        torch.cuda.current_stream(model.device).wait_event(dt.ready)
        counts = self.transport.all_gather(dt.hist).cpu().numpy().astype(np.int64)  # (G, L, K)
        local = _LocalTable(counts, self.rank, self.kl)
        plan = plan_placement(local, self.state, budget, eb)
        for g in plan.groups:
            if any(k[0] == g.layer and k[1] in local.required_by_layer()[g.layer]
                   for k in g.evictions):
                raise UnservableError("a layer's local expert working set exceeds the budget")
        issuer = _GroupIssuer(self, plan, local.required_by_layer())
        if getattr(self.transport, "peer", False):
            return self._forward_peer(table, dt, counts, issuer, lengths, tokens_dev)
        # per-layer regroup maps and local offsets, uploaded once per batch
        maps = [ep_regroup(counts, l, self.rank, self.world) for l in range(c.num_layers)]
        splits = [ep_splits(counts, l, self.rank, self.world) for l in range(c.num_layers)]
        k = dt.k
        with torch.cuda.stream(cs):
            cs.wait_event(dt.ready)
            dt.use_on(cs)
            lay = BatchLayout(list(lengths), tokens_dev, model.device)
            x = model.embed_layout(lay)
            xb = None
            n_rows = x.shape[0] * k
            for layer in range(c.num_layers):
                done = issuer.issue_for(layer)
                x = model.attention_mix(layer, x, lay, xb=xb)
                off_t, perm, alpha_perm = dt.layer(layer)
                x_perm = torch.empty((n_rows, c.d_model), dtype=torch.bfloat16, device=x.device)
                _lib.check(h.sida_gather_rows_bf16(x.data_ptr(), perm.data_ptr(), n_rows, k,
                                                   c.d_model, x_perm.data_ptr(), cs.cuda_stream))
                send_rows, recv_rows = splits[layer]
                recv = self.transport.all_to_all(x_perm, send_rows, recv_rows)
                src, off_local = maps[layer]
                n_recv = int(src.size)
                y_recv = torch.empty((n_recv, c.d_model), dtype=torch.bfloat16, device=x.device)
                if n_recv:
                    src_t = torch.from_numpy(src).pin_memory().to(x.device, non_blocking=True)
                    off_l = torch.from_numpy(off_local).pin_memory().to(x.device, non_blocking=True)
                    x_loc = torch.empty((n_recv, c.d_model), dtype=torch.bfloat16, device=x.device)
                    _lib.check(h.sida_gather_bf16_rows(recv.data_ptr(), src_t.data_ptr(), n_recv,
                                                       c.d_model, x_loc.data_ptr(), cs.cuda_stream))
                    row = issuer.slot_row(layer)
                    row_t = torch.from_numpy(row).pin_memory().to(x.device, non_blocking=True)
                    hidden = torch.empty((n_recv, c.expert_hidden), dtype=torch.bfloat16,
                                         device=x.device)
                    if done is not None:
                        cs.wait_event(done)
                    _lib.check(h.sida_grouped_ffn_bf16(
                        x_loc.data_ptr(), n_recv, c.d_model, c.expert_hidden, off_l.data_ptr(),
                        self.kl, row_t.data_ptr(), None, 0, store.base_ptr, store.slot_stride,
                        store.n_slots, src_t.data_ptr(), None, None, None, y_recv.data_ptr(),
                        hidden.data_ptr(), store.err_flag.data_ptr(), cs.cuda_stream))
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    store.mark_read(row, ev)
                y_back = self.transport.all_to_all(y_recv, recv_rows, send_rows)
                out = torch.empty_like(x)
                xb = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
                _lib.check(h.sida_unpermute_combine(
                    y_back.data_ptr(), dt.inv[layer].data_ptr(), alpha_perm.data_ptr(),
                    x.data_ptr(), x.shape[0], k, c.d_model, out.data_ptr(), xb.data_ptr(),
                    cs.cuda_stream))
                x = out
            logits = model.pool_classify(x, lay)
        return logits

    # ------------------------------------------------------------------ peer memory
    def _forward_peer(self, table, dt, counts, issuer, lengths, tokens_dev):
        """The EP layer with both exchanges fused into the producing epilogues
        (PeerTransport): out-projection → owners' receive buffers (by layer
        parity) → flags → local grouped FFN whose GEMM2 epilogue writes into
        the sources' return buffers → flags → unpermute-combine."""
        model, store, budget, tp = self.model, self.store, self.budget, self.transport
        c = model.config
        h = _lib.lib()
        eb = model.expert_bytes_each()
        cs = self.base.compute_stream
        k = dt.k
        n_rows = int(sum(lengths)) * k
        rows_max = int(counts.sum(axis=2).max())  # largest (token, rank) count of any source
        if not tp.ready or rows_max > tp.cap_y:
            tp.setup(model, max(rows_max, getattr(tp, "cap_y", 0)) * 2)
        dev = model.device

        def h2d(a):
            return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)

        with torch.cuda.stream(cs):
            cs.wait_event(dt.ready)
            dt.use_on(cs)
            lay = BatchLayout(list(lengths), tokens_dev, dev)
            x = model.embed_layout(lay)
            xb = None
            for layer in range(c.num_layers):
                done = issuer.issue_for(layer)
                d_start, d_val, r_start, r_val, off_l, n_recv = ep_peer_maps(
                    counts, layer, self.rank, self.world, tp.cap_x, tp.cap_y)
                d_start_t, d_val_t = h2d(d_start), h2d(d_val)
                dmap = torch.empty(n_rows, dtype=torch.int32, device=dev)
                _lib.check(h.sida_segment_map(d_start_t.data_ptr(), d_val_t.data_ptr(), c.num_experts,
                                              dt.inv[layer].data_ptr(), n_rows, dmap.data_ptr(),
                                              cs.cuda_stream))
                par = layer & 1
                x_attn = model.attention_mix(layer, x, lay, xb=xb,
                                             scatter=("peer", dmap, k, tp.xloc_peers[par],
                                                      tp.cap_x))
                tp.exchange_done(cs)  # every source's rows are in my receive buffer
                if n_recv:
                    r_start_t, r_val_t = h2d(r_start), h2d(r_val)
                    rmap = torch.empty(n_recv, dtype=torch.int32, device=dev)
                    _lib.check(h.sida_segment_map(r_start_t.data_ptr(), r_val_t.data_ptr(),
                                                  self.kl * self.world, None, n_recv,
                                                  rmap.data_ptr(), cs.cuda_stream))
                    row = issuer.slot_row(layer)
                    row_t, off_t = h2d(row), h2d(off_l)
                    hidden = torch.empty((n_recv, c.expert_hidden), dtype=torch.bfloat16,
                                         device=dev)
                    if done is not None:
                        cs.wait_event(done)
                    _lib.check(h.sida_grouped_ffn_bf16_peer(
                        tp.xloc[par].data_ptr(), n_recv, c.d_model, c.expert_hidden,
                        off_t.data_ptr(), self.kl, row_t.data_ptr(), store.base_ptr,
                        store.slot_stride, store.n_slots, rmap.data_ptr(), tp.yback_peers.data_ptr(),
                        tp.cap_y, hidden.data_ptr(), store.err_flag.data_ptr(), cs.cuda_stream))
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    store.mark_read(row, ev)
                tp.exchange_done(cs)  # every owner's outputs are in my return buffer
                _, _, alpha_perm = dt.layer(layer)
                out = torch.empty_like(x_attn)
                xb = torch.empty(x_attn.shape, dtype=torch.bfloat16, device=dev)
                _lib.check(h.sida_unpermute_combine(
                    tp.yback.data_ptr(), dt.inv[layer].data_ptr(), alpha_perm.data_ptr(),
                    x_attn.data_ptr(), x_attn.shape[0], k, c.d_model, out.data_ptr(),
                    xb.data_ptr(), cs.cuda_stream))
                x = out
            logits = model.pool_classify(x, lay)
        return logits
