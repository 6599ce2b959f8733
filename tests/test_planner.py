"""Native residency planner (csrc/planner.cpp via offload.plan_placement)
against the reference's own plans (tests/golden/planner.json) and against the
oracle restatement on randomized multi-batch workloads (ref
tests/test_offload.py:150-170 style, state-for-state)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import offload as ooff
from paper_2310_18859_b200.errors import ContractError, UnservableError
from paper_2310_18859_b200.offload import (
    MemoryBudget,
    ResidencyState,
    apply_plan,
    effective_utilization,
    plan_placement,
)


class FakeTable:
    def __init__(self, layers):
        self.layers = [set(s) for s in layers]

    def required_by_layer(self):
        return self.layers

    def required_experts(self):
        return {(l, e) for l, s in enumerate(self.layers) for e in s}


def test_replays_reference_plans():
    cases = json.load(open(os.path.join(GOLDEN, "planner.json")))
    for case in cases:
        eb = case["expert_bytes"]
        budget = MemoryBudget(case["slots"] * eb, bandwidth_bytes_per_s=case["bandwidth"],
                              per_transfer_latency_s=case["latency"])
        state = ResidencyState()
        for b in case["batches"]:
            plan = plan_placement(FakeTable(b["required"]), state, budget, eb)
            assert len(plan.groups) == len(b["groups"])
            for mine, ref in zip(plan.groups, b["groups"]):
                assert [[op, list(k)] for op, k in mine.steps] == ref["steps"]
                assert mine.prefetchable == ref["prefetchable"]
                assert mine.transfer_s == pytest.approx(ref["transfer_s"], rel=1e-12)
            state, secs = apply_plan(state, plan)
            assert secs == pytest.approx(b["seconds"], rel=1e-12)
            assert [list(k) for k in state.fifo_order] == b["fifo_after"]


def test_random_workload_matches_oracle_state_for_state():
    g = np.random.default_rng(11)
    eb = 7
    for trial in range(60):
        L, K = int(g.integers(1, 6)), int(g.integers(1, 12))
        slots = int(g.integers(1, L * K + 3))
        budget = MemoryBudget(slots * eb)
        state = ResidencyState()
        res, fifo, used = {}, [], 0
        for _ in range(int(g.integers(1, 20))):
            req = [set(g.integers(0, K, size=int(g.integers(0, K + 1))).tolist()) for _ in range(L)]
            plan = plan_placement(FakeTable(req), state, budget, eb)
            ref = ooff.plan(req, res, fifo, used, slots * eb, eb)
            assert [g_.steps for g_ in plan.groups] == [r["steps"] for r in ref]
            assert [g_.prefetchable for g_ in plan.groups] == [r["prefetchable"] for r in ref]
            for r in ref:
                used = ooff.apply_group(res, fifo, used, r, slots * eb, eb)
            state, _ = apply_plan(state, plan)
            assert state.fifo_order == fifo
            assert state.used_bytes <= slots * eb


def test_full_budget_never_evicts():
    req = [{0, 1, 2}, {0, 3}, {1}]
    plan = plan_placement(FakeTable(req), ResidencyState(), MemoryBudget(100 * 10), 10)
    assert plan.evictions == [] and len(plan.loads) == 6


def test_within_layer_swap_is_not_prefetchable():
    plan = plan_placement(FakeTable([{0, 1, 2}]), ResidencyState(), MemoryBudget(20), 10)
    assert plan.groups[0].prefetchable is False
    assert plan.evictions == [(0, 0)]


def test_unservable_and_contract_errors():
    with pytest.raises(UnservableError):
        plan_placement(FakeTable([{0}]), ResidencyState(), MemoryBudget(5), 10)
    state = ResidencyState({(0, 1): 3}, [(0, 1)], 3)
    with pytest.raises(ContractError):
        plan_placement(FakeTable([{0}]), state, MemoryBudget(100), 10)
    plan = plan_placement(FakeTable([{0}]), ResidencyState(), MemoryBudget(100), 10)
    other = ResidencyState({(0, 5): 10}, [(0, 5)], 10)
    with pytest.raises(ContractError):
        apply_plan(other, plan)


def test_effective_utilization():
    state = ResidencyState({(0, 1): 10, (0, 2): 10}, [(0, 1), (0, 2)], 20)
    assert effective_utilization(state, {(0, 1)}) == 0.5
    with pytest.raises(ContractError):
        effective_utilization(state, {(1, 1)})


# ------------------------------------------------------------- spread victim policy
class _Uniform:
    def __init__(self, L, K, drop=()):
        self.L, self.K, self.drop = L, K, set(drop)

    def required_by_layer(self):
        return [{e for e in range(self.K) if (l, e) not in self.drop} for l in range(self.L)]


@pytest.mark.parametrize("slots", [86, 72, 48, 20])
def test_spread_policy_plans_are_valid_and_spread(slots):
    """plan_placement_spread (opt-in, not the reference's plan): every group
    applies within the budget, every layer's experts are resident when it
    runs, no group evicts an expert its own layer needs unless the layer alone
    exceeds the budget, and at 86 of 96 slots the steady state is one load per
    layer (the reference FIFO plan: 12-18 loads clustered on the first layers)."""
    from paper_2310_18859_b200.offload import (MemoryBudget, ResidencyState,
                                               apply_group_inplace, plan_placement_spread)

    L, K = 12, 8
    st = ResidencyState()
    rng = np.random.default_rng(slots)
    for j in range(8):
        drop = {(int(l), int(e)) for l, e in zip(rng.integers(0, L, 3), rng.integers(0, K, 3))} \
            if j % 2 else ()
        table = _Uniform(L, K, drop)
        req = table.required_by_layer()
        plan = plan_placement_spread(table, st, MemoryBudget(slots), 1)
        for g in plan.groups:
            for k in g.evictions:
                assert not (k[0] == g.layer and k[1] in req[g.layer])
            apply_group_inplace(st, g, slots, 1)
            assert st.used_bytes <= slots
            assert all((g.layer, e) in st.resident for e in req[g.layer])
        st.check()
    if slots == 86:  # back to uniform routing: settles at <= 12 loads, <= 2 per layer
        for _ in range(4):
            plan = plan_placement_spread(_Uniform(L, K), st, MemoryBudget(slots), 1)
            for g in plan.groups:
                apply_group_inplace(st, g, slots, 1)
        loads = [len(g.loads) for g in plan.groups]
        assert sum(loads) <= 12 and max(loads) <= 2, loads
        assert all(g.prefetchable for g in plan.groups)


@pytest.mark.parametrize("slots", [1, 3, 7])
def test_spread_policy_tiny_budgets(slots):
    """Budgets below one layer's working set (multi-wave layers): the spread
    planner evicts the layer's own earlier loads like the FIFO planner's class
    4, stays within the budget and loads every required expert."""
    from paper_2310_18859_b200.offload import (MemoryBudget, ResidencyState,
                                               apply_group_inplace, plan_placement_spread)

    st = ResidencyState()
    table = _Uniform(2, 8)
    for _ in range(3):
        plan = plan_placement_spread(table, st, MemoryBudget(slots), 1)
        for g in plan.groups:
            assert sorted(k[1] for k in g.loads) == sorted(
                e for e in range(8) if (g.layer, e) not in st.resident)
            apply_group_inplace(st, g, slots, 1)
            assert st.used_bytes <= slots
        st.check()


def test_spread_policy_uses_the_next_batch_table():
    """Hash-driven victims (plan_placement_spread(..., next_table=...)): with a
    skewed stream whose hot experts recur batch after batch and a budget that
    holds the hot set plus a little, knowing the next batch's table cuts the
    expert loads, and an expert the next batch needs is never evicted while an
    expert neither batch needs is resident."""
    from paper_2310_18859_b200.offload import (MemoryBudget, ResidencyState,
                                               apply_group_inplace, plan_placement_spread)

    L, K, slots = 6, 32, 6 * 20
    rng = np.random.default_rng(7)
    hot = [set(rng.choice(K, 14, replace=False).tolist()) for _ in range(L)]
    stream = []
    for _ in range(12):
        layers = []
        for layer in range(L):
            cold = set(rng.choice(K, 6, replace=False).tolist())
            layers.append(hot[layer] | cold)
        stream.append(FakeTable(layers))

    def run(aware):
        st = ResidencyState()
        loads = 0
        for j, table in enumerate(stream):
            nxt = stream[j + 1] if aware and j + 1 < len(stream) else None
            plan = plan_placement_spread(table, st, MemoryBudget(slots), 1, next_table=nxt)
            req = table.required_by_layer()
            for g in plan.groups:
                if nxt is not None:
                    nreq = nxt.required_by_layer()
                    live = set(st.resident)
                    for op, k in g.steps:
                        if op == "load":
                            live.add(k)
                            continue
                        live.discard(k)
                        if k[1] in nreq[k[0]] and k[1] not in req[k[0]]:
                            # a next-batch expert went while an unneeded one stayed?
                            assert not any(e not in req[l] and e not in nreq[l]
                                           for (l, e) in live)
                apply_group_inplace(st, g, slots, 1)
                loads += len(g.loads) if j >= 2 else 0
            st.check()
        return loads

    blind, aware = run(False), run(True)
    assert aware < blind, (aware, blind)
