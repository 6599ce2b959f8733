"""Expert parallelism across the GPUs of one box.

Rank r owns experts [r*K/G, (r+1)*K/G) of every MoE layer (contiguous blocks),
holds only those in its HBM slot arena, and serves its own batch stream
(hash, embed and attention are local). Per batch the ranks exchange their
(L, K) expert histograms once -- SiDA knows every layer's routing before
inference starts, so there is no per-layer size handshake -- and every map
of the batch is derived from that count matrix: segment tables on the host
(O(G K) per layer, vectorised, one pinned upload per batch), row-level maps
on the device (`sida_segment_map`). Per layer, with the local experts split
into C chunks:

  send    = out-proj epilogue scatter   each token's bf16 expert input goes
            straight to its dispatch position (chunk-major, then destination
            rank, expert, token): no gather pass
  recv_c  = all_to_all(send_c)          NCCL, one per chunk, all issued at once
  x_loc_c = regroup(recv_c)             (source, expert) -> expert-major
  ret_c   = grouped FFN (chunk c experts); the GEMM2 epilogue writes each row
            back to its receive position as bf16 (row_map)
  back_c  = all_to_all(ret_c)           issued right after FFN c
  out     = x_attn + sum_r alpha * back sida_map_combine (ranks in order)

The collectives run on NCCL's stream, so dispatch c+1 overlaps FFN c and
return c overlaps FFN c+1. `GlooTransport` stages the same data path through
host memory (tests: several ranks on one GPU or CPU-only hosts);
`PeerTransport` replaces both exchanges with epilogue stores into peer
memory.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .errors import ContractError, UnservableError
from .moe import BatchLayout, MoEModel
from .offload import (
    ExpertStore,
    MemoryBudget,
    ResidencyState,
    apply_group_inplace,
    plan_placement,
    plan_placement_spread,
)
from .predictor import DeviceTableRing


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
    """Receive buffer (source-major, then local expert) -> expert-major order
    (the host oracle of the device-built regroup map, one chunk).

    Returns (src (R,) int32: receive position of each expert-major row,
    off (Kl+1,) int32 expert offsets of the expert-major rows)."""
    kl = owner_block(counts.shape[2], world)
    c = counts[:, layer, rank * kl:(rank + 1) * kl].astype(np.int64)  # (G, Kl)
    starts = np.concatenate([[0], np.cumsum(c.reshape(-1))[:-1]]).reshape(world, kl)
    per_e = c.sum(axis=0)
    off = np.zeros(kl + 1, dtype=np.int32)
    np.cumsum(per_e, out=off[1:])
    src = np.empty(int(per_e.sum()), dtype=np.int32)
    for e in range(kl):
        pos = off[e]
        for g in range(world):
            n = int(c[g, e])
            src[pos:pos + n] = np.arange(starts[g, e], starts[g, e] + n, dtype=np.int32)
            pos += n
    return src, off


def chunk_bounds(kl: int, chunks: int) -> np.ndarray:
    """Local-expert boundaries of the C exchange chunks (contiguous blocks)."""
    c = max(1, min(chunks, kl))
    return np.array([(i * kl) // c for i in range(c + 1)], dtype=np.int64)


def ep_layer_plan(counts: np.ndarray, layer: int, rank: int, world: int, chunks: int) -> dict:
    """Segment tables and split sizes of one layer of the chunked NCCL path,
    from the (G, L, K) count matrix (vectorised numpy).

    dispatch: my rows in x_perm (expert-sorted) order are laid out chunk-major
      (chunk c, then owner q, then expert, then token) in the send buffer;
      expert e's rows start at d_val[e] (segments d_start = my expert offsets);
    chunk c: send_rows[q] / recv_rows[g]; the receive buffer is source-major
      (g, then local expert); regroup segments (x_loc order, expert-major /
      source-minor) map each x_loc row to its receive position; off_local
      (kc + 1) delimit the chunk's local experts in x_loc; n_recv rows."""
    G = world
    c = counts[:, layer, :].astype(np.int64)                   # (G, K)
    K = c.shape[1]
    kl = owner_block(K, G)
    b = chunk_bounds(kl, chunks)
    C = len(b) - 1
    mine = c[rank]
    off_me = np.zeros(K + 1, dtype=np.int64)
    np.cumsum(mine, out=off_me[1:])
    # block (chunk ci, owner q) = experts q*kl + [b[ci], b[ci+1]), contiguous in x_perm
    first = np.array([[q * kl + b[ci] for q in range(G)] for ci in range(C)])      # (C, G)
    last = np.array([[q * kl + b[ci + 1] for q in range(G)] for ci in range(C)])
    sizes = off_me[last] - off_me[first]                                          # (C, G)
    dstart = np.concatenate([[0], np.cumsum(sizes.reshape(-1))[:-1]]).reshape(C, G)
    e = np.arange(K)
    q_of, el_of = e // kl, e % kl
    ci_of = np.searchsorted(b, el_of, side="right") - 1
    d_val = dstart[ci_of, q_of] + (off_me[e] - off_me[first[ci_of, q_of]])
    chunk_rows = sizes.sum(axis=1)
    out = {"d_start": off_me[:K].astype(np.int32), "d_val": d_val.astype(np.int32),
           "chunk_start": np.concatenate([[0], np.cumsum(chunk_rows)]).astype(np.int64),
           "chunks": []}
    lo = rank * kl
    for ci in range(C):
        cc = c[:, lo + b[ci]:lo + b[ci + 1]]                   # (G, kc) rows from each source
        kc = cc.shape[1]
        rs = np.concatenate([[0], np.cumsum(cc.reshape(-1))[:-1]]).reshape(G, kc)   # recv (g, el)
        ccT = cc.T                                                                     # (kc, G)
        xs = np.concatenate([[0], np.cumsum(ccT.reshape(-1))[:-1]]).reshape(kc, G)  # x_loc (el, g)
        per_e = cc.sum(axis=0)
        off_l = np.zeros(kc + 1, dtype=np.int64)
        np.cumsum(per_e, out=off_l[1:])
        out["chunks"].append({
            "experts": (int(b[ci]), int(b[ci + 1])),
            "send_rows": sizes[ci].tolist(), "recv_rows": cc.sum(axis=1).tolist(),
            "seg_start": xs.reshape(-1).astype(np.int32),
            "seg_val": rs.T.reshape(-1).astype(np.int32),
            "off_local": off_l.astype(np.int32), "n_recv": int(off_l[-1])})
    return out


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

    def all_to_all(self, send: torch.Tensor, send_rows, recv_rows,
                   recv: torch.Tensor | None = None) -> torch.Tensor:
        recv, wait = self.all_to_all_async(send, send_rows, recv_rows, recv)
        wait()
        return recv

    def all_to_all_async(self, send, send_rows, recv_rows, recv=None):
        """Enqueue the exchange (it waits for the current stream's work) and
        return (recv, wait) -- wait() makes the current stream wait for it."""
        if recv is None:
            recv = torch.empty((int(sum(recv_rows)),) + tuple(send.shape[1:]), dtype=send.dtype,
                               device=send.device)
        work = dist.all_to_all_single(recv, send, output_split_sizes=[int(v) for v in recv_rows],
                                      input_split_sizes=[int(v) for v in send_rows],
                                      group=self.group, async_op=True)
        return recv, work.wait


class GlooTransport(NcclTransport):
    """Same interface, staged through host memory (gloo collectives)."""

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        h = t.detach().cpu().contiguous()
        world = dist.get_world_size(self.group)
        parts = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(parts, h, group=self.group)
        return torch.stack(parts).to(t.device)

    def all_to_all_async(self, send, send_rows, recv_rows, recv=None):
        hs = send.detach().cpu().contiguous()
        raw = hs.view(torch.uint8).reshape(hs.shape[0], -1)  # gloo moves raw bytes per row
        got = torch.empty((int(sum(recv_rows)), raw.shape[1]), dtype=torch.uint8)
        dist.all_to_all_single(got, raw, output_split_sizes=[int(v) for v in recv_rows],
                               input_split_sizes=[int(v) for v in send_rows], group=self.group)
        out = got.view(send.dtype).reshape((-1,) + tuple(send.shape[1:])).to(send.device)
        if recv is not None:
            recv.copy_(out)
            out = recv
        return out, (lambda: None)


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
    """SiDA serving with experts sharded over the ranks of ``group``; the
    same interface as `engine.SidaEngine` (hash_tokens / forward / check_errors,
    hash + compute + copy streams), so `serve_sida(..., engine=...)` drives it.

    Residency is per rank over its own expert block (the reference planner on
    the union of every rank's needs for those experts). A layer whose local
    working set exceeds the budget is rejected (waves are single-GPU only).
    ``chunks``: exchange chunks per layer (NCCL path)."""

    def __init__(self, model: MoEModel, predictor, budget: MemoryBudget, transport=None,
                 group=None, eval_top_k: int = 1, victim_policy: str = "fifo", chunks: int = 2):
        from .engine import SidaEngine  # streams + hash plumbing

        if victim_policy not in ("fifo", "spread"):
            raise ContractError(f"unknown victim policy {victim_policy!r}")
        self.model = model
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.kl = owner_block(model.config.num_experts, self.world)
        self.transport = transport or NcclTransport(group)
        self.base = SidaEngine(model, predictor, budget, eval_top_k)
        self.hash_stream = self.base.hash_stream
        self.compute_stream = self.base.compute_stream
        self.store: ExpertStore = self.base.store
        self.state = ResidencyState()
        self.budget = budget
        self.victim_policy = victim_policy
        self.chunks = max(1, int(chunks))
        self.peak = 0
        self.ffn_events = None  # (per-layer FFN timing is single-GPU only)
        self.mix_events: list = []

    def hash_tokens(self, batch_id, tokens_dev, lengths):
        """Hash + permute on the hash stream, then this batch's histogram
        all-gather enqueued right away (every rank hashes its batches in the
        same order, so the collectives match): by the time `forward` needs the
        count matrix it has long arrived, and the gather never queues behind
        the previous batch's exchanges."""
        table = self.base.hash_tokens(batch_id, tokens_dev, lengths)
        table._ep_counts = self._gather_counts(table._dev)
        return table

    def check_errors(self, tables=(), extra_flags=()) -> None:
        self.base.check_errors(tables, extra_flags)

    def _gather_counts(self, dt):
        """(G, L, K) histograms of every rank's batch: one all-gather per
        batch, enqueued behind the hash stream (not the busy compute stream),
        copied to pinned host memory; returns (host tensor, ready event)."""
        with torch.cuda.stream(self.hash_stream):
            self.hash_stream.wait_event(dt.ready)
            g = self.transport.all_gather(dt.hist)
            host = torch.empty(g.shape, dtype=g.dtype, pin_memory=True)
            host.copy_(g, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.hash_stream)
        return host, ev

    def _counts(self, table, dt) -> np.ndarray:
        pend = getattr(table, "_ep_counts", None)
        host, ev = pend if pend is not None else self._gather_counts(dt)
        ev.synchronize()
        return host.numpy().astype(np.int64)

    def forward(self, table, lengths, tokens_dev=None, batch=None, next_table=None):
        """One batch; returns (logits (n_seq, C) on the device, record dict,
        (start, end) events on the compute stream) like SidaEngine.forward."""
        model, budget = self.model, self.budget
        eb = model.expert_bytes_each()
        cs = self.compute_stream
        dt = table.on_device(model, stream=self.hash_stream)
        if tokens_dev is None:
            tokens_dev = dt.tokens_for(model, batch, cs)
        counts = self._counts(table, dt)
        local = _LocalTable(counts, self.rank, self.kl)
        planner = plan_placement if self.victim_policy == "fifo" else plan_placement_spread
        plan = planner(local, self.state, budget, eb)
        for g in plan.groups:
            if any(k[0] == g.layer and k[1] in local.required_by_layer()[g.layer]
                   for k in g.evictions):
                raise UnservableError("a layer's local expert working set exceeds the budget")
        issuer = _GroupIssuer(self, plan, local.required_by_layer())
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        cs.wait_event(dt.ready)
        dt.use_on(cs)
        ev0.record(cs)
        if getattr(self.transport, "peer", False):
            logits = self._forward_peer(dt, counts, issuer, lengths, tokens_dev)
        else:
            logits = self._forward_nccl(dt, counts, issuer, lengths, tokens_dev)
        ev1.record(cs)
        DeviceTableRing.release(table, cs)
        resident_req = [k for k in local.required_experts() if k in self.state.resident]
        util = (sum(self.state.resident[k] for k in resident_req) / self.state.used_bytes
                if self.state.used_bytes else 1.0)
        rec = {"batch_id": table.batch_id, "num_samples": len(lengths),
               "num_tokens": int(sum(lengths)), "transfer_s": plan.estimated_transfer_s,
               "expert_loads": len(plan.loads), "groups_issued_ahead": 0, "utilization": util}
        return logits, rec, (ev0, ev1)

    # ------------------------------------------------------------------ NCCL, chunked
    @staticmethod
    def _upload_plans(plans, dev):
        """Every segment table of the batch in one pinned H2D copy."""
        parts, index = [], []
        pos = 0

        def add(a):
            nonlocal pos
            parts.append(np.asarray(a, dtype=np.int32))
            index.append((pos, len(a)))
            pos += len(a)
            return len(index) - 1

        keys = []
        for p in plans:
            k = {"d_start": add(p["d_start"]), "d_val": add(p["d_val"]), "chunks": []}
            for ch in p["chunks"]:
                k["chunks"].append({n: add(ch[n]) for n in ("seg_start", "seg_val", "off_local")})
            keys.append(k)
        flat = np.concatenate(parts) if parts else np.zeros(1, dtype=np.int32)
        buf = torch.from_numpy(flat).pin_memory().to(dev, non_blocking=True)

        def view(i):
            a, n = index[i]
            return buf[a:a + n]

        out = [{"d_start": view(k["d_start"]), "d_val": view(k["d_val"]),
                "chunks": [{n: view(i) for n, i in ch.items()} for ch in k["chunks"]]}
               for k in keys]
        return out, buf

    def _forward_nccl(self, dt, counts, issuer, lengths, tokens_dev):
        model, store, tp = self.model, self.store, self.transport
        c = model.config
        h = _lib.lib()
        cs = self.compute_stream
        sh = cs.cuda_stream
        k = dt.k
        d = c.d_model
        dev = model.device
        plans = [ep_layer_plan(counts, l, self.rank, self.world, self.chunks)
                 for l in range(c.num_layers)]
        with torch.cuda.stream(cs):
            dplans, _buf = self._upload_plans(plans, dev)
            lay = BatchLayout(list(lengths), tokens_dev, dev)
            x, xb = model.embed_layout(lay, with_bf16=True)
            n_rows = x.shape[0] * k
            for layer in range(c.num_layers):
                done = issuer.issue_for(layer)
                pl, dpl = plans[layer], dplans[layer]
                # dispatch positions of my (token, rank) rows (chunk-major)
                dmap = torch.empty(n_rows, dtype=torch.int32, device=dev)
                _lib.check(h.sida_segment_map(dpl["d_start"].data_ptr(), dpl["d_val"].data_ptr(),
                                              c.num_experts, dt.inv[layer].data_ptr(), n_rows,
                                              dmap.data_ptr(), sh))
                send = torch.empty((n_rows, d), dtype=torch.bfloat16, device=dev)
                x_attn = model.attention_mix(layer, x, lay, xb=xb, scatter=(dmap, k, send))
                back = torch.empty((n_rows, d), dtype=torch.bfloat16, device=dev)
                cstart = pl["chunk_start"]
                recvs = [tp.all_to_all_async(send[cstart[i]:cstart[i + 1]], ch["send_rows"],
                                             ch["recv_rows"])
                         for i, ch in enumerate(pl["chunks"])]
                row = issuer.slot_row(layer)
                row_t = store.rows.upload(row, cs)
                if done is not None:
                    cs.wait_event(done)
                waits = []
                for i, (ch, dch) in enumerate(zip(pl["chunks"], dpl["chunks"])):
                    recv, wait = recvs[i]
                    wait()
                    n_recv = ch["n_recv"]
                    ret = torch.empty((n_recv, d), dtype=torch.bfloat16, device=dev)
                    e0, e1 = ch["experts"]
                    if n_recv:
                        src = torch.empty(n_recv, dtype=torch.int32, device=dev)
                        _lib.check(h.sida_segment_map(
                            dch["seg_start"].data_ptr(), dch["seg_val"].data_ptr(),
                            (e1 - e0) * self.world, None, n_recv, src.data_ptr(), sh))
                        x_loc = torch.empty((n_recv, d), dtype=torch.bfloat16, device=dev)
                        _lib.check(h.sida_gather_bf16_rows(recv.data_ptr(), src.data_ptr(),
                                                           n_recv, d, x_loc.data_ptr(), sh))
                        hidden = torch.empty((n_recv, c.expert_hidden), dtype=torch.bfloat16,
                                             device=dev)
                        _lib.check(h.sida_grouped_ffn_bf16(
                            x_loc.data_ptr(), n_recv, d, c.expert_hidden,
                            dch["off_local"].data_ptr(), e1 - e0, row_t[e0:e1].data_ptr(), None,
                            0, store.base_ptr, store.slot_stride, store.n_slots, src.data_ptr(),
                            None, None, None, ret.data_ptr(), hidden.data_ptr(),
                            store.err_flag.data_ptr(), sh))
                    _, w = tp.all_to_all_async(ret, ch["recv_rows"], ch["send_rows"],
                                               back[cstart[i]:cstart[i + 1]])
                    waits.append(w)
                ev = torch.cuda.Event()
                ev.record(cs)
                store.mark_read(row, ev)
                for w in waits:
                    w()
                out = torch.empty_like(x_attn)
                xb = torch.empty(x_attn.shape, dtype=torch.bfloat16, device=dev)
                _lib.check(h.sida_map_combine(back.data_ptr(), dmap.data_ptr(),
                                              dt.alpha_f32[layer].data_ptr(), x_attn.data_ptr(),
                                              x_attn.shape[0], k, d, out.data_ptr(),
                                              xb.data_ptr(), sh))
                x = out
            logits = model.pool_classify(x, lay)
        return logits

    # ------------------------------------------------------------------ peer memory
    def _forward_peer(self, dt, counts, issuer, lengths, tokens_dev):
        """The EP layer with both exchanges fused into the producing epilogues
        (PeerTransport): out-projection → owners' receive buffers (by layer
        parity) → flags → local grouped FFN whose GEMM2 epilogue writes into
        the sources' return buffers → flags → unpermute-combine."""
        model, store, tp = self.model, self.store, self.transport
        c = model.config
        h = _lib.lib()
        cs = self.compute_stream
        k = dt.k
        n_rows = int(sum(lengths)) * k
        rows_max = int(counts.sum(axis=2).max())  # largest (token, rank) count of any source
        if not tp.ready or rows_max > tp.cap_y:
            tp.setup(model, max(rows_max, getattr(tp, "cap_y", 0)) * 2)
        dev = model.device

        def h2d(a):
            return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)

        with torch.cuda.stream(cs):
            lay = BatchLayout(list(lengths), tokens_dev, dev)
            x, xb = model.embed_layout(lay, with_bf16=True)
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
