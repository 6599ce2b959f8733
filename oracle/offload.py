"""FIFO residency planner restatement (oracle; test infrastructure only).

Restates ref `pkg/src/sida/offload.py`: `plan_placement` (`:118-140`),
the four victim classes (`_victim_class`, `:143-152`), the per-layer group
builder (`_plan_groups`, `:155-204`) including the `prefetchable` rule
(`:179-183`) and the linear transfer-cost model (`:192-195`), and
`apply_group_inplace` (`:207-222`) and the reactive single-layer load of
standard serving, `ensure_layer_resident` (`:240-278`).

State is (resident: dict[(layer, expert)] -> bytes, fifo: list of keys in
arrival order, used: int). A plan is a list of groups
``{"layer", "steps": [("evict"|"load", (l, e))...], "prefetchable", "transfer_s"}``.
"""

from __future__ import annotations


class Unservable(RuntimeError):
    pass


def victim_class(key, planning_layer: int, required) -> int:
    """1: not needed by this batch; 2: needed only by an earlier layer;
    3: needed by a later layer; 4: needed by the layer being planned."""
    lay, e = key
    if not (lay < len(required) and e in required[lay]):
        return 1
    if lay < planning_layer:
        return 2
    return 3 if lay > planning_layer else 4


def plan(required, resident: dict, fifo: list, used: int, budget_bytes: int,
         expert_bytes: int, bandwidth: float = 16e9, latency: float = 50e-6):
    """Returns the list of per-layer groups; does not mutate the inputs."""
    if expert_bytes > budget_bytes:
        raise Unservable("expert larger than the budget")
    res = dict(resident)
    order = list(fifo)
    groups = []
    for layer, need in enumerate(required):
        missing = [(layer, e) for e in sorted(need) if (layer, e) not in res]
        steps = []
        prefetchable = True
        for key in missing:
            while used + expert_bytes > budget_bytes:
                best = None
                for cand in order:
                    cls = victim_class(cand, layer, required)
                    if best is None or cls < best[0]:
                        best = (cls, cand)
                        if cls == 1:
                            break
                if best is None:
                    raise Unservable("nothing evictable while over budget")
                cls, victim = best
                if cls == 4 or (cls == 2 and victim[0] == layer - 1):
                    prefetchable = False
                used -= res.pop(victim)
                order.remove(victim)
                steps.append(("evict", victim))
            res[key] = expert_bytes
            order.append(key)
            used += expert_bytes
            steps.append(("load", key))
        n = len(missing)
        groups.append(dict(layer=layer, steps=steps, prefetchable=prefetchable,
                           transfer_s=n * expert_bytes / bandwidth + latency * n))
    return groups


def apply_group(resident: dict, fifo: list, used: int, group, budget_bytes: int,
                expert_bytes: int) -> int:
    """Mutates (resident, fifo); returns the new used-bytes total."""
    for op, key in group["steps"]:
        if op == "evict":
            if key not in resident:
                raise ValueError(f"plan/state mismatch: evicting non-resident {key}")
            used -= resident.pop(key)
            fifo.remove(key)
        else:
            if key in resident:
                raise ValueError(f"plan/state mismatch: loading resident {key}")
            if used + expert_bytes > budget_bytes:
                raise ValueError("plan exceeds budget mid-application")
            resident[key] = expert_bytes
            fifo.append(key)
            used += expert_bytes
    return used


def ensure_layer(resident: dict, fifo: list, used: int, layer: int, expert_ids,
                 budget_bytes: int, expert_bytes: int):
    """ref `offload.py:240-278`: evict FIFO among residents the layer does not
    need (else the FIFO head), then load the missing experts in ascending
    order. Mutates (resident, fifo); returns (steps, used)."""
    if expert_bytes > budget_bytes:
        raise Unservable("expert larger than the budget")
    req = {int(e) for e in expert_ids}
    loads = [(layer, e) for e in sorted(req) if (layer, e) not in resident]
    steps = []
    for key in loads:
        while used + expert_bytes > budget_bytes:
            victim = next((c for c in fifo if not (c[0] == layer and c[1] in req)), fifo[0])
            used -= resident.pop(victim)
            fifo.remove(victim)
            steps.append(("evict", victim))
        resident[key] = expert_bytes
        fifo.append(key)
        used += expert_bytes
        steps.append(("load", key))
    return steps, used
