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
import time

import numpy as np
import torch

from .errors import ContractError, UnservableError
from .moe import BatchLayout, MoEModel
from .offload import (
    ExpertStore,
    MemoryBudget,
    ResidencyState,
    Wave,
    apply_group_inplace,
    plan_placement,
    run_waves,
)
from .predictor import ExpertHashTable, hash_device


def prepare_waves(plan, required, store: ExpertStore) -> list[list[Wave]]:
    """Slot bookkeeping for a whole plan, in plan order. A group that evicts
    an expert of its own layer (victim class 4, ref offload.py:14-16) is split
    into waves: each wave's FFN runs over the layer's experts resident at that
    point, before the eviction reuses their slots."""
    out = []
    for g in plan.groups:
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
        out.append(waves)
    return out


class SidaEngine:
    """Streams, HBM slot arena and residency state of one serving instance."""

    def __init__(self, model: MoEModel, predictor, budget: MemoryBudget, eval_top_k: int = 1,
                 prefetch: str = "layer", store: ExpertStore | None = None, streams=None):
        if prefetch not in ("layer", "batch"):
            raise ContractError(f"unknown prefetch mode {prefetch!r}")
        if model.expert_bytes_each() > budget.fast_tier_bytes:
            raise UnservableError("budget cannot hold a single expert")
        self.model = model
        self.predictor = predictor
        self.budget = budget
        self.eval_top_k = eval_top_k
        self.prefetch = prefetch
        dev = model.device
        # compute at the highest stream priority: the persistent GEMM grids get
        # SMs first; the hash (one batch ahead) fills what is left
        lo, hi = torch.cuda.Stream.priority_range()
        if os.environ.get("SIDA_FLAT_PRIORITY"):  # A/B switch for measurements
            lo = hi = 0
        self.hash_stream, self.compute_stream = streams or (
            torch.cuda.Stream(device=dev, priority=lo), torch.cuda.Stream(device=dev, priority=hi))
        if os.environ.get("SIDA_HASH_SERIAL") and streams is None:  # A/B: one stream
            self.hash_stream = self.compute_stream
        self.store = store or ExpertStore.for_budget(model, budget)
        self.state = getattr(self.store, "residency_state", None) or ResidencyState()
        self.store.residency_state = self.state
        self.peak = 0
        self.ffn_events: list | None = None  # set to a list to time every layer's FFN
        self.mix_events: list = []           # (filled alongside ffn_events) attention_mix

    # -- hash stream ------------------------------------------------------------------
    def hash_tokens(self, batch_id: int, tokens_dev: torch.Tensor, lengths) -> ExpertHashTable:
        """Hash + permute for device-resident tokens on the hash stream."""
        return hash_device(self.predictor, self.model, tokens_dev, list(lengths),
                           self.eval_top_k, batch_id, self.hash_stream)

    # -- compute stream ---------------------------------------------------------------
    def forward(self, table: ExpertHashTable, lengths, tokens_dev: torch.Tensor | None = None,
                batch=None):
        """Run one batch; returns (logits (n_seq, C) on the device, record dict,
        (start_event, end_event) on the compute stream)."""
        model, store, state, budget = self.model, self.store, self.state, self.budget
        eb = model.expert_bytes_each()
        n_layers = model.config.num_layers
        cs = self.compute_stream
        required = table.required_by_layer()
        if len(required) < n_layers:
            raise ContractError(f"missing hash entry for (layer {len(required)}, token 0)")
        plan = plan_placement(table, state, budget, eb)
        waves = prepare_waves(plan, required, store)
        dt = table.on_device(model, stream=self.hash_stream)
        if tokens_dev is None:
            tokens_dev = dt.tokens_for(model, batch)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        cs.wait_event(dt.ready)
        dt.use_on(cs)
        ev0.record(cs)
        done: list = [None] * n_layers
        issued = [False] * n_layers

        def issue(idx: int):
            apply_group_inplace(state, plan.groups[idx], budget.fast_tier_bytes, eb)
            issued[idx] = True
            self.peak = max(self.peak, state.used_bytes)
            if len(waves[idx]) == 1:
                done[idx] = store.enqueue_loads(waves[idx][0].loads)

        if self.prefetch == "batch":
            # every group whose victims are not read by this batch's earlier layers
            for idx, g in enumerate(plan.groups):
                safe = len(waves[idx]) == 1 and all(
                    not (k[0] < idx and k[1] in required[k[0]]) for k in g.evictions)
                if safe and all(issued[:idx]):
                    issue(idx)
        with torch.cuda.stream(cs):
            lay = BatchLayout(list(lengths), tokens_dev, model.device)
            x = model.embed_layout(lay)
            xb = None  # bf16 copy of x for the next attention GEMM (FFN epilogue output)
            for layer in range(n_layers):
                if not issued[layer]:
                    issue(layer)
                if (self.prefetch == "layer" and layer + 1 < n_layers
                        and plan.groups[layer + 1].prefetchable and not issued[layer + 1]):
                    issue(layer + 1)
                if self.ffn_events is not None:
                    e_m = torch.cuda.Event(enable_timing=True)
                    e_m.record(cs)
                scatter = None
                if model.wo_t is not None and dt.k <= 4:
                    x_perm = torch.empty((lay.n_tokens * dt.k, model.config.d_model),
                                         dtype=torch.bfloat16, device=x.device)
                    scatter = (dt.inv[layer], dt.k, x_perm)
                x = model.attention_mix(layer, x, lay, xb=xb, scatter=scatter)
                xp = scatter[2] if scatter is not None else None
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
            logits = model.pool_classify(x, lay)
        ev1.record(cs)
        resident_req = [k for k in table.required_experts() if k in state.resident]
        util = (sum(state.resident[k] for k in resident_req) / state.used_bytes
                if state.used_bytes else 1.0)
        record = {
            "batch_id": table.batch_id,
            "num_samples": len(lengths),
            "num_tokens": int(sum(lengths)),
            "transfer_s": plan.estimated_transfer_s,
            "expert_loads": len(plan.loads),
            "utilization": util,
        }
        return logits, record, (ev0, ev1)
