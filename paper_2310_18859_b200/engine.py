"""One batch of SiDA serving on the compute stream (shared by serve_sida and
the device-resident bench path).

`SidaEngine.forward` is the body of the reference's inference worker
(ref pipeline.py:217-289) for one dequeued table: plan placement
(`plan_placement`), slot bookkeeping for every group (`prepare_waves`), then
per layer -- issue the layer's load group if not yet issued, issue the next
layer's group when it is prefetchable (ref pipeline.py:246-253), run the
mixing attention, wait for this layer's copies only, run the grouped FFN --
and finally the classifier head. Nothing here blocks the host on the GPU
except the (L x K) histogram the planner needs, which was produced by the
hash stream one batch ahead.
"""

from __future__ import annotations

import os

import torch

from .errors import ContractError, UnservableError
from .moe import BatchLayout, MoEModel
from .offload import (
    FFN_SLOT_MSG,
    OUTPROJ_MSG,
    PERMUTE_MSG,
    ExpertStore,
    MemoryBudget,
    ResidencyState,
    Wave,
    apply_group_inplace,
    check_device_flags,
    plan_placement,
    plan_placement_spread,
    run_waves,
)
from .predictor import DeviceTableRing, ExpertHashTable


def prepare_waves(plan, required, store: ExpertStore) -> list[list[Wave]]:
    """Slot bookkeeping for a whole plan, in plan order. A group that evicts
    an expert of its own layer (victim class 4, ref offload.py:14-16) is split
    into waves: each wave's FFN runs over the layer's experts resident at that
    point, before the eviction reuses their slots."""
    return [prepare_group_waves(g, required, store) for g in plan.groups]


def prepare_group_waves(g, required, store: ExpertStore) -> list[Wave]:
    """Slot bookkeeping of one group (groups must be prepared in plan order)."""
    layer = g.layer
    need = sorted(required[layer])
    waves, loads, done = [], [], set()
    for op, key in g.steps:
        if op == "evict":
            if key[0] == layer and key[1] in required[layer]:
                exp = [e for e in need if (layer, e) in store.slot_of and e not in done]
                waves.append(Wave(layer, loads, exp, store.slot_row(layer, exp)))
                done.update(exp)
                loads = []
            store.free_slot(key)
        else:
            loads.append((key, store.take_slot(key)))
    exp = [e for e in need if e not in done]
    waves.append(Wave(layer, loads, exp, store.slot_row(layer, exp)))
    return waves


def multi_wave(g, required) -> bool:
    """A group that evicts an expert its own layer needs runs in waves."""
    return any(k[0] == g.layer and k[1] in required[g.layer] for k in g.evictions)


class _BatchPlan:
    """Placement plan of one batch plus its issue state (groups issued, copy
    done-events), so a batch can be planned and partly issued while the
    previous one is still computing."""

    def __init__(self, table, required, plan, waves):
        self.table = table
        self.required = required
        self.plan = plan
        self.waves = waves  # per group, prepared (slot bookkeeping) when issued
        n = len(plan.groups)
        self.issued = [False] * n
        self.done: list = [None] * n
        self.early = 0  # groups issued before this batch's forward started


class _StaticTable:
    """The per-layer permutation arrays a captured forward reads."""

    def __init__(self, dt):
        self.k = dt.k
        self.off, self.perm = dt.off.clone(), dt.perm.clone()
        self.inv, self.alpha_perm = dt.inv.clone(), dt.alpha_perm.clone()

    def layer(self, layer: int):
        return self.off[layer], self.perm[layer], self.alpha_perm[layer]


class _GraphEntry:
    """One captured forward for a fixed lengths signature: static token and
    permutation buffers, per-layer expert -> slot rows on the device, the
    graph and its logits buffer (graph-private memory pool)."""

    def __init__(self, eng: "SidaEngine", lengths, dt, tokens_dev, waves):
        model, cs = eng.model, eng.compute_stream
        self.tokens = tokens_dev.clone()
        self.table = _StaticTable(dt)
        self.lay = BatchLayout(list(lengths), self.tokens, model.device)
        self.row_host = [w[0].slot_row.copy() for w in waves]
        self.rows = [eng.store.rows.upload(r, cs).clone() for r in self.row_host]
        # one eager pass first (library handles, lazily loaded kernels), then capture
        eng._graph_body(self.lay, self.table, waves, self.rows)
        # (capture_begin/end directly: torch.cuda.graph() would also run a
        # full gc.collect() and empty the caching allocator on every capture)
        self.graph = torch.cuda.CUDAGraph()
        cs.synchronize()
        with torch.cuda.stream(cs):
            self.graph.capture_begin(capture_error_mode="thread_local")
            try:
                self.logits = eng._graph_body(self.lay, self.table, waves, self.rows)
            finally:
                self.graph.capture_end()

    def load(self, dt, tokens_dev, waves, store, cs) -> None:
        t = self.table
        self.tokens.copy_(tokens_dev, non_blocking=True)
        for dst, src in ((t.off, dt.off), (t.perm, dt.perm), (t.inv, dt.inv),
                         (t.alpha_perm, dt.alpha_perm)):
            dst.copy_(src, non_blocking=True)
        for layer, w in enumerate(waves):
            r = w[0].slot_row
            if len(r) != len(self.row_host[layer]) or (r != self.row_host[layer]).any():
                self.rows[layer][: len(r)].copy_(store.rows.upload(r, cs))
                self.row_host[layer] = r.copy()


class SidaEngine:
    """Streams, HBM slot arena and residency state of one serving instance."""

    def __init__(self, model: MoEModel, predictor, budget: MemoryBudget, eval_top_k: int = 1,
                 prefetch: str = "layer", store: ExpertStore | None = None, streams=None,
                 victim_policy: str = "fifo"):
        if prefetch not in ("layer", "batch"):
            raise ContractError(f"unknown prefetch mode {prefetch!r}")
        # "fifo": the reference planner (bit-identical plans); "spread": the
        # opt-in victim order of offload.plan_placement_spread
        if victim_policy not in ("fifo", "spread"):
            raise ContractError(f"unknown victim policy {victim_policy!r}")
        self.victim_policy = victim_policy
        if model.expert_bytes_each() > budget.fast_tier_bytes:
            raise UnservableError("budget cannot hold a single expert")
        self.model = model
        self.predictor = predictor
        self.budget = budget
        self.eval_top_k = eval_top_k
        self.prefetch = prefetch
        dev = model.device
        # hash and compute streams at the same priority: measured at the bench
        # shape (tools/pipe_ab.py, base-128, 32K tokens) 8.84-8.97 ms per step
        # against 9.57-10.35 ms with the compute stream prioritised (the starved
        # hash kernels then land on SMs late and hold back whole persistent GEMM
        # grids) and 9.74-9.83 ms with the hash serialised on the compute stream.
        # SIDA_STREAM_PRIORITY=1 restores the prioritised arrangement (A/B).
        lo = hi = 0
        if os.environ.get("SIDA_STREAM_PRIORITY") == "1":
            lo, hi = torch.cuda.Stream.priority_range()
        self.hash_stream, self.compute_stream = streams or (
            torch.cuda.Stream(device=dev, priority=lo), torch.cuda.Stream(device=dev, priority=hi))
        if os.environ.get("SIDA_HASH_SERIAL") and streams is None:  # A/B: one stream
            self.hash_stream = self.compute_stream
        self.store = store or ExpertStore.for_budget(model, budget)
        self.state = getattr(self.store, "residency_state", None) or ResidencyState()
        self.store.residency_state = self.state
        self.peak = 0
        self.ffn_events: list | None = None  # set to a list to time every layer's FFN
        self.trace: list | None = None       # set to a list: (name, stream, ev0, ev1) timeline
        self.mix_events: list = []           # (filled alongside ffn_events) attention_mix
        # hash-driven cross-batch prefetch: during the last `lookahead` layers
        # of batch j, the (already hashed) batch j+1 is planned and its leading
        # load groups are issued; forward(j+1) picks the plan up from here
        self.lookahead = int(os.environ.get("SIDA_XBATCH_LOOKAHEAD", "0"))
        # prefetch depth in layers: group g may be issued during layer l < g
        # when none of its victims is read by layers l..g (reference: 1)
        self.depth = int(os.environ.get("SIDA_PREFETCH_DEPTH", "1"))
        self._pending: _BatchPlan | None = None
        # CUDA-graph replay of whole forwards (see _forward_graph): batches of
        # at most `graph_max_tokens` tokens whose experts are all resident; a
        # lengths signature is captured the second time it is seen
        self.graph_max_tokens = int(os.environ.get("SIDA_GRAPH_MAX_TOKENS", "16384"))
        self.graph_cap = 8
        self._graphs: dict = {}
        self._graph_seen: dict = {}
        self.graph_replays = 0
        # device table ring behind hash_tokens (one batch hashed ahead + slack)
        self.ring = DeviceTableRing(3, dev, strict=False)

    # -- hash stream ------------------------------------------------------------------
    def _mark(self, stream):
        if self.trace is None:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        return ev

    def hash_tokens(self, batch_id: int, tokens_dev: torch.Tensor, lengths) -> ExpertHashTable:
        """Hash + permute for device-resident tokens on the hash stream, into
        the next slot of the engine's device table ring (forward releases it;
        with three tables outstanding, or ids out of order, the table is built
        in fresh allocations instead)."""
        t0 = self._mark(self.hash_stream)
        table = self.ring.produce(self.predictor, self.model, lengths, self.eval_top_k,
                                  self.hash_stream, batch_id, tokens_dev=tokens_dev)
        if t0 is not None:
            self.trace.append((f"hash+permute b{batch_id}", "hash", t0,
                               self._mark(self.hash_stream)))
        return table

    # -- compute stream ---------------------------------------------------------------
    def forward(self, table: ExpertHashTable, lengths, tokens_dev: torch.Tensor | None = None,
                batch=None, next_table: ExpertHashTable | None = None):
        """Run one batch; returns (logits (n_seq, C) on the device, record dict,
        (start_event, end_event) on the compute stream). ``next_table`` (the
        next batch's hash table, if already built) enables the cross-batch
        prefetch of `_issue_ahead`."""
        model, store, state, budget = self.model, self.store, self.state, self.budget
        eb = model.expert_bytes_each()
        n_layers = model.config.num_layers
        cs = self.compute_stream
        bp = self._pending if (self._pending is not None and self._pending.table is table) \
            else self._plan_batch(table, next_table)
        self._pending = None
        required, plan, waves = bp.required, bp.plan, bp.waves
        dt = table.on_device(model, stream=self.hash_stream)
        if tokens_dev is None:
            tokens_dev = dt.tokens_for(model, batch, cs)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        cs.wait_event(dt.ready)
        dt.use_on(cs)
        ev0.record(cs)
        done, issued = bp.done, bp.issued
        if self._graphable(bp, dt, lengths):
            logits = self._forward_graph(bp, dt, lengths, tokens_dev)
            ev1.record(cs)
            DeviceTableRing.release(table, cs)
            return logits, self._record(table, lengths, bp), (ev0, ev1)

        def issue(idx: int):
            self._issue(bp, idx)

        if self.prefetch == "batch":
            # every group whose victims are not read by this batch's earlier layers
            for idx, g in enumerate(plan.groups):
                safe = not multi_wave(g, required) and all(
                    not (k[0] < idx and k[1] in required[k[0]]) for k in g.evictions)
                if safe and all(issued[:idx]):
                    issue(idx)
        with torch.cuda.stream(cs):
            lay = BatchLayout(list(lengths), tokens_dev, model.device)
            # x fp32 residual stream, xb its bf16 copy for the next QKV GEMM
            # (written by the embedding kernel, then by each FFN epilogue)
            x, xb = model.embed_layout(lay, with_bf16=True)
            for layer in range(n_layers):
                if not issued[layer]:
                    issue(layer)
                if (self.prefetch == "layer" and layer + 1 < n_layers
                        and plan.groups[layer + 1].prefetchable and not issued[layer + 1]):
                    issue(layer + 1)
                if self.prefetch == "layer":
                    for g_idx in range(layer + 2, min(n_layers, layer + 1 + self.depth)):
                        if issued[g_idx]:
                            continue
                        g = plan.groups[g_idx]
                        if (not all(issued[:g_idx]) or multi_wave(g, required)
                                or any(layer <= k[0] <= g_idx for k in g.evictions)):
                            break
                        issue(g_idx)
                if (next_table is not None and self._pending is None
                        and layer >= n_layers - self.lookahead and all(issued)):
                    self._issue_ahead(next_table, bp, layer)
                if self.ffn_events is not None:
                    e_m = torch.cuda.Event(enable_timing=True)
                    e_m.record(cs)
                scatter = None
                if model.wo_t is not None and dt.k <= 4:
                    x_perm = torch.empty((lay.n_tokens * dt.k, model.config.d_model),
                                         dtype=torch.bfloat16, device=x.device)
                    scatter = (dt.inv[layer], dt.k, x_perm)
                t_a = self._mark(cs)
                x = model.attention_mix(layer, x, lay, xb=xb, scatter=scatter)
                xp = scatter[2] if scatter is not None else None
                t_f = self._mark(cs)
                if self.ffn_events is not None:
                    e_a = torch.cuda.Event(enable_timing=True)
                    e_a.record(cs)
                    self.mix_events.append((e_m, e_a))
                xb = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
                if len(waves[layer]) == 1:
                    x = run_waves(model, waves[layer], x, dt, store, cs, pre_done=[done[layer]],
                                  out_bf16=xb, x_perm=xp)
                else:
                    x = run_waves(model, waves[layer], x, dt, store, cs,
                                  issue=lambda w: store.enqueue_loads(w.loads), out_bf16=xb,
                                  x_perm=xp)
                if self.ffn_events is not None:
                    e_b = torch.cuda.Event(enable_timing=True)
                    e_b.record(cs)
                    self.ffn_events.append((e_a, e_b, x.shape[0], len(required[layer])))
                if t_a is not None:
                    t_e = self._mark(cs)
                    self.trace.append((f"attention L{layer}", "compute", t_a, t_f))
                    self.trace.append((f"ffn L{layer} (waits own copies)", "compute", t_f, t_e))
            logits = model.pool_classify(x, lay)
        ev1.record(cs)
        DeviceTableRing.release(table, cs)
        return logits, self._record(table, lengths, bp), (ev0, ev1)

    def _record(self, table, lengths, bp: _BatchPlan) -> dict:
        state, plan = self.state, bp.plan
        resident_req = [k for k in table.required_experts() if k in state.resident]
        util = (sum(state.resident[k] for k in resident_req) / state.used_bytes
                if state.used_bytes else 1.0)
        return {
            "batch_id": table.batch_id,
            "num_samples": len(lengths),
            "num_tokens": int(sum(lengths)),
            "transfer_s": plan.estimated_transfer_s,
            "expert_loads": len(plan.loads),
            "groups_issued_ahead": bp.early,
            "utilization": util,
        }

    def check_errors(self, tables=(), extra_flags=()) -> None:
        """Raise ContractError if a kernel flagged a contract violation since
        the last check (synchronises; call where the host already waits):
        the FFN / out-projection flags, the ring slots' sticky permute flags,
        and those of ``tables`` built outside a ring."""
        flags = [(FFN_SLOT_MSG, self.store.err_flag), (OUTPROJ_MSG, self.model._err)]
        flags += [(PERMUTE_MSG, f) for f in list(self.ring.error_flags()) + list(extra_flags)]
        for t in tables:
            dt = getattr(t, "_dev", None)
            if dt is not None and getattr(t, "_slot", None) is None:
                flags.append((PERMUTE_MSG, dt.err))
        check_device_flags(flags)

    # -- CUDA-graph replay ---------------------------------------------------------------
    def _graphable(self, bp: _BatchPlan, dt, lengths) -> bool:
        """Small batches are host-bound (~0.2 ms of Python + launches per
        layer against a few us of GPU work), so a forward that moves no
        expert runs as one graph launch. Eligible: no copies in the plan (all
        required experts resident), single-wave layers, the fused
        out-projection path, no per-layer timing requested."""
        n_tok = int(sum(lengths))
        if (n_tok > self.graph_max_tokens or self.ffn_events is not None
                or self.model.wo_t is None or dt.k > 4 or bp.plan.loads):
            return False
        key = (tuple(int(n) for n in lengths), dt.k)
        if key not in self._graphs:
            self._graph_seen[key] = self._graph_seen.get(key, 0) + 1
            if self._graph_seen[key] < 2:
                return False  # one-off shapes stay eager
        for idx in range(len(bp.plan.groups)):
            if not bp.issued[idx]:
                self._issue(bp, idx)  # bookkeeping only: the plan has no loads
        return all(len(w) == 1 for w in bp.waves)

    def _graph_body(self, lay: BatchLayout, dt, waves, rows):
        model, cs = self.model, self.compute_stream
        x, xb = model.embed_layout(lay, with_bf16=True)
        for layer in range(model.config.num_layers):
            x_perm = torch.empty((lay.n_tokens * dt.k, model.config.d_model),
                                 dtype=torch.bfloat16, device=x.device)
            x = model.attention_mix(layer, x, lay, xb=xb, scatter=(dt.inv[layer], dt.k, x_perm))
            xb = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
            x = run_waves(model, waves[layer], x, dt, self.store, cs, out_bf16=xb,
                          x_perm=x_perm, rows_dev=[rows[layer]])
        return model.pool_classify(x, lay)

    def _forward_graph(self, bp: _BatchPlan, dt, lengths, tokens_dev):
        """Copy the batch's tokens and permutation into the graph's static
        buffers, refresh any expert -> slot row that changed, replay. The
        slots read are marked with one event after the replay."""
        cs, store = self.compute_stream, self.store
        key = (tuple(int(n) for n in lengths), dt.k)
        ent = self._graphs.pop(key, None)
        with torch.cuda.stream(cs):
            if ent is None:
                ent = _GraphEntry(self, lengths, dt, tokens_dev, bp.waves)
                if len(self._graphs) >= self.graph_cap:
                    self._graphs.pop(next(iter(self._graphs)))
            else:
                ent.load(dt, tokens_dev, bp.waves, store, cs)
            self._graphs[key] = ent  # most recently used last
            ent.graph.replay()
            logits = ent.logits.clone()
        ev = torch.cuda.Event()
        ev.record(cs)
        for w in bp.waves:
            store.mark_read(w[0].slot_row, ev)
        self.graph_replays += 1
        return logits

    # -- planning / issue ---------------------------------------------------------------
    def _plan_batch(self, table, next_table=None) -> _BatchPlan:
        """ref pipeline.py:217-225: plan against the residency state left by
        every group issued so far, and do the slot bookkeeping of all groups.
        The spread policy also reads the next batch's table when it is built
        (hash-driven victims: experts neither batch needs go first)."""
        n_layers = self.model.config.num_layers
        required = table.required_by_layer()
        if len(required) < n_layers:
            raise ContractError(f"missing hash entry for (layer {len(required)}, token 0)")
        if self.victim_policy == "fifo":
            plan = plan_placement(table, self.state, self.budget, self.model.expert_bytes_each())
        else:
            nt = next_table if next_table is not None and self._table_ready(next_table) else None
            plan = plan_placement_spread(table, self.state, self.budget,
                                         self.model.expert_bytes_each(), next_table=nt)
        return _BatchPlan(table, required, plan, [None] * len(plan.groups))

    @staticmethod
    def _table_ready(table) -> bool:
        """Host tables always; device tables once their hash (and histogram)
        has completed -- planning never waits on the hash stream."""
        dt = getattr(table, "_dev", None)
        return dt is None or (dt.hist is not None and dt.ready.query())

    def _issue(self, bp: _BatchPlan, idx: int) -> None:
        """ref pipeline.py:229-235 issue(): apply the group to the residency
        state and enqueue its copies (single-wave groups; multi-wave groups
        copy just in time inside run_waves)."""
        g = bp.plan.groups[idx]
        apply_group_inplace(self.state, g, self.budget.fast_tier_bytes,
                            self.model.expert_bytes_each())
        bp.waves[idx] = prepare_group_waves(g, bp.required, self.store)
        bp.issued[idx] = True
        self.peak = max(self.peak, self.state.used_bytes)
        if len(bp.waves[idx]) == 1:
            bp.done[idx] = self.store.enqueue_loads(bp.waves[idx][0].loads)

    def _issue_ahead(self, next_table, bp: _BatchPlan, layer: int) -> None:
        """Hash-driven cross-batch prefetch. Batch j+1's table is known while
        batch j computes (SiDA builds tables one batch ahead), so once every
        group of batch j is issued its plan can be made and its leading groups
        issued now: a group goes early only if it is single-wave, prefetchable
        (or the first), and evicts nothing batch j still reads in layers >=
        `layer`. Copies into reused slots still wait on the slot's last
        reader, so they overlap batch j's remaining layers."""
        dtn = getattr(next_table, "_dev", None)
        if dtn is not None and (dtn.hist is None or not dtn.ready.query()):
            return  # not hashed yet: never block the compute loop on it
        n_layers = self.model.config.num_layers
        remaining = {(l, e) for l in range(layer, n_layers) for e in bp.required[l]}
        nbp = self._plan_batch(next_table)
        for idx, g in enumerate(nbp.plan.groups):
            if multi_wave(g, nbp.required) or (idx > 0 and not g.prefetchable):
                break
            if any(k in remaining for k in g.evictions):
                break
            self._issue(nbp, idx)
            nbp.early += 1
        self._pending = nbp
