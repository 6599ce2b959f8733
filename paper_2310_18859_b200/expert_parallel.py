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
            tokens_dev = dt.tokens_for(model, batch)
        torch.cuda.current_stream(model.device).wait_event(dt.ready)
        counts = self.transport.all_gather(dt.hist).cpu().numpy().astype(np.int64)  # (G, L, K)
        local = _LocalTable(counts, self.rank, self.kl)
        plan = plan_placement(local, self.state, budget, eb)
        for g in plan.groups:
            if any(k[0] == g.layer and k[1] in local.required_by_layer()[g.layer]
                   for k in g.evictions):
                raise UnservableError("a layer's local expert working set exceeds the budget")
        loads_by_layer = []
        for g in plan.groups:
            ls = []
            for op, key in g.steps:
                if op == "evict":
                    store.free_slot(key)
                else:
                    ls.append((key, store.take_slot(key)))
            loads_by_layer.append(ls)
        # per-layer regroup maps and local offsets, uploaded once per batch
        lo_e = self.rank * self.kl
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
                apply_group_inplace(self.state, plan.groups[layer], budget.fast_tier_bytes, eb)
                self.peak = max(self.peak, self.state.used_bytes)
                done = store.enqueue_loads(loads_by_layer[layer])
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
                    row = np.full(self.kl, -1, dtype=np.int32)
                    for e in range(self.kl):
                        key = (layer, lo_e + e)
                        if key in store.slot_of:
                            row[e] = store.slot_of[key]
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
