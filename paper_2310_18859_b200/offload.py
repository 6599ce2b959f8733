"""Expert residency: the reference planner API over a real HBM slot arena.

Mirrors ref pkg/src/sida/offload.py (`MemoryBudget`, `ResidencyState`,
`PlanGroup`, `PlacementPlan`, `plan_placement`, `apply_group_inplace`,
`apply_plan`, `ensure_layer_resident`, `effective_utilization`,
`memory_reduction`). Decisions come
from the native planner (`sida_plan_placement`, csrc/planner.cpp) and are
identical to the reference's FIFO victim classes; `ExpertStore` executes them
for real: one HBM arena of ``n_slots`` expert slots, pinned host expert
images, and `cudaMemcpyAsync` copies on a dedicated copy stream, each
ordered after the last kernel that read the slot it overwrites (the
simulated `time.sleep` transfers of ref pipeline.py:141-146 become real
copies overlapped with the previous layer's compute).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ContractError, UnservableError

Key = tuple[int, int]  # (layer, expert id)


@dataclass
class MemoryBudget:
    """ref offload.py:36-46. ``fast_tier_bytes`` is the HBM expert budget;
    the bandwidth/latency pair only feeds the reported cost model."""

    fast_tier_bytes: int
    bandwidth_bytes_per_s: float = 16e9
    per_transfer_latency_s: float = 50e-6

    def __post_init__(self):
        if self.bandwidth_bytes_per_s <= 0:
            raise ContractError("bandwidth must be positive")
        if self.fast_tier_bytes < 0:
            raise ContractError("fast tier budget must be non-negative")


@dataclass
class ResidencyState:
    """ref offload.py:49-67."""

    resident: dict = field(default_factory=dict)
    fifo_order: list = field(default_factory=list)
    used_bytes: int = 0

    def copy(self) -> "ResidencyState":
        return ResidencyState(dict(self.resident), list(self.fifo_order), self.used_bytes)

    def fingerprint(self) -> tuple:
        return (tuple(self.fifo_order), self.used_bytes)

    def check(self) -> None:
        if sorted(self.fifo_order) != sorted(self.resident):
            raise ContractError("fifo_order is not a permutation of resident")
        if self.used_bytes != sum(self.resident.values()):
            raise ContractError("used_bytes does not match resident sizes")


@dataclass
class PlanGroup:
    """ref offload.py:70-91."""

    layer: int
    steps: list
    prefetchable: bool
    transfer_s: float

    @property
    def loads(self) -> list:
        return [k for op, k in self.steps if op == "load"]

    @property
    def evictions(self) -> list:
        return [k for op, k in self.steps if op == "evict"]


@dataclass
class PlacementPlan:
    """ref offload.py:94-111."""

    groups: list
    budget_bytes: int
    expert_bytes: int
    source_fingerprint: tuple

    @property
    def loads(self) -> list:
        return [k for g in self.groups for k in g.loads]

    @property
    def evictions(self) -> list:
        return [k for g in self.groups for k in g.evictions]

    @property
    def estimated_transfer_s(self) -> float:
        return sum(g.transfer_s for g in self.groups)


def plan_placement(table, state: ResidencyState, budget: MemoryBudget,
                   expert_bytes: int) -> PlacementPlan:
    """Per-layer load/evict groups (ref offload.py:118-140), computed by the
    native planner. ``table`` is anything with ``required_by_layer()``."""
    if expert_bytes > budget.fast_tier_bytes:
        raise UnservableError(
            f"expert of {expert_bytes} bytes exceeds budget {budget.fast_tier_bytes}")
    required = table.required_by_layer()
    n_layers = len(required)
    keys = state.fifo_order
    sizes = set(state.resident.values())
    if (sizes and sizes != {expert_bytes}) or len(keys) != len(state.resident):
        raise ContractError("residency state holds experts of another size")
    kv = np.array(keys, dtype=np.int64).reshape(-1, 2)
    max_e = max([max(s) for s in required if s] + [int(kv[:, 1].max()) if len(kv) else 0, 0])
    K = max_e + 1
    req = np.zeros((max(n_layers, 1), K), dtype=np.uint8)
    for layer, s in enumerate(required):
        if s:
            req[layer, np.fromiter(s, dtype=np.int64, count=len(s))] = 1
    fifo = (kv[:, 0] * K + kv[:, 1]).astype(np.int32)
    cap = 2 * n_layers * K + len(keys) + 1
    steps = np.empty(cap, dtype=np.int32)
    goff = np.empty(n_layers + 1, dtype=np.int32)
    pref = np.empty(max(n_layers, 1), dtype=np.uint8)
    budget_slots = budget.fast_tier_bytes // expert_bytes
    _lib.check(_lib.load().sida_plan_placement(
        req.ctypes.data, n_layers, K, int(budget_slots), fifo.ctypes.data, len(keys),
        steps.ctypes.data, cap, goff.ctypes.data, pref.ctypes.data))
    groups = []
    for layer in range(n_layers):
        raw = steps[goff[layer] : goff[layer + 1]]
        st = [("load", divmod(int(v), K)) if v >= 0 else ("evict", divmod(int(-v - 1), K))
              for v in raw]
        n_loads = int(np.count_nonzero(raw >= 0))
        groups.append(PlanGroup(
            layer=layer, steps=st, prefetchable=bool(pref[layer]),
            transfer_s=n_loads * expert_bytes / budget.bandwidth_bytes_per_s
            + budget.per_transfer_latency_s * n_loads))
    return PlacementPlan(groups=groups, budget_bytes=budget.fast_tier_bytes,
                         expert_bytes=expert_bytes, source_fingerprint=state.fingerprint())


def plan_placement_spread(table, state: ResidencyState, budget: MemoryBudget,
                          expert_bytes: int, next_table=None) -> PlacementPlan:
    """Opt-in victim policy (no reference counterpart; ``SidaEngine(...,
    victim_policy="spread")``): the same per-layer groups as
    ``plan_placement`` -- loads are the layer's missing experts in ascending
    order -- with victims chosen to keep the next batch's misses spread over
    the layers. Preference: not needed by this batch; consumed by a layer
    before the previous one (the group stays prefetchable); needed later in
    this batch; the previous layer's; the planned layer's own (multi-wave).
    Within a class the layer that has given up the fewest experts to this plan
    goes first, then the furthest next use, then arrival order.

    The reference's FIFO classes evict the oldest consumed experts, so with
    uniform routing and a budget below the working set a batch's loads pile
    onto its first layers (Switch-base-8 at 86 of 96 slots: 15.3 loads per
    batch, 8/2/6/2 on layers 0-3) and a layer's copies outlast the compute
    they could hide behind. Spread victims settle at one load per layer (12
    per batch) there, and at 1-3 per layer at 72 slots, each within a
    layer's compute when issued a layer ahead.

    ``next_table`` (the next batch's hash table, which SiDA has already built
    while this batch is planned): among the experts this batch does not need,
    those the next batch does not need either go first -- the hash-driven
    half of the victim order. Without it the order is as above."""
    if expert_bytes > budget.fast_tier_bytes:
        raise UnservableError(
            f"expert of {expert_bytes} bytes exceeds budget {budget.fast_tier_bytes}")
    required = table.required_by_layer()
    n_layers = len(required)
    keys = list(state.fifo_order)
    n_keys = len(keys)
    n_missing = sum(len(r) for r in required)
    cap = n_keys + n_missing + 1
    # resident keys in arrival order (loads appended), as arrays for one
    # vectorised argmin per eviction
    kl = np.zeros(cap, dtype=np.int64)
    ke = np.zeros(cap, dtype=np.int64)
    if n_keys:
        kv = np.array(keys, dtype=np.int64).reshape(-1, 2)
        kl[:n_keys], ke[:n_keys] = kv[:, 0], kv[:, 1]
    alive = np.zeros(cap, dtype=bool)
    alive[:n_keys] = True
    n_pos = n_keys
    max_e = max([max(r) for r in required if r] + [int(ke[:n_keys].max()) if n_keys else 0, 0])
    req = np.zeros((max(n_layers, int(kl[:n_keys].max()) + 1 if n_keys else 0, 1), max_e + 1),
                   dtype=bool)
    for layer, r in enumerate(required):
        if r:
            req[layer, np.fromiter(r, dtype=np.int64, count=len(r))] = True
    nxt = None
    if next_table is not None:
        nreq = next_table.required_by_layer()
        nxt = np.zeros_like(req)
        for layer, r in enumerate(nreq):
            r = [e for e in r if e < req.shape[1]]
            if r and layer < req.shape[0]:
                nxt[layer, np.asarray(r, dtype=np.int64)] = True
    resident = set(keys)
    used = state.used_bytes
    budget_bytes = budget.fast_tier_bytes
    taken = np.zeros(req.shape[0], dtype=np.int64)
    pos_all = np.arange(cap, dtype=np.int64)
    groups = []
    for layer in range(n_layers):
        need = required[layer]
        missing = [(layer, e) for e in sorted(need) if (layer, e) not in resident]
        steps = []
        prefetchable = True
        cand = None  # per-group candidate arrays, rebuilt only when they run dry
        for key in missing:
            while used + expert_bytes > budget_bytes:
                if cand is not None and not cand[5].any():
                    # only when one layer's experts exceed the budget (multi-wave):
                    # this group's own loads become candidates (class 4)
                    cand = None
                if cand is None:
                    idx = np.nonzero(alive[:n_pos])[0]
                    ll = kl[idx]
                    needed = req[ll, ke[idx]]
                    cls = np.where(~needed, 0,
                                   np.where(ll == layer, 4,
                                            np.where(ll < layer - 1, 1,
                                                     np.where(ll > layer, 2, 3))))
                    # (class 0 split by the next batch's table: its experts
                    # are evicted after the ones neither batch needs)
                    nx = nxt[ll, ke[idx]] if nxt is not None else np.zeros(idx.size, bool)
                    dist = np.where(ll < layer, n_layers - layer + ll, ll - layer)
                    # (class, evictions already taken from the layer, furthest
                    # next use, arrival order) as one lexicographic integer key
                    hi = (cls * 2 + (nx & (cls == 0))) * 4096
                    lo = (255 - np.clip(dist, 0, 255)) * 65536 + pos_all[idx]
                    free = np.ones(idx.size, dtype=bool)
                    cand = (idx, ll, cls, hi, lo, free)
                idx, ll, cls, hi, lo, free = cand
                score = (hi + np.minimum(taken[ll], 4095)) * (256 * 65536) + lo
                score[~free] = np.iinfo(np.int64).max
                i = int(np.argmin(score))
                if not free[i]:
                    raise UnservableError("nothing evictable while over budget")
                free[i] = False
                j = int(idx[i])
                vcls = int(cls[i])
                victim = (int(kl[j]), int(ke[j]))
                if vcls >= 3:
                    prefetchable = False
                taken[victim[0]] += 1
                alive[j] = False
                resident.discard(victim)
                used -= expert_bytes
                steps.append(("evict", victim))
            kl[n_pos], ke[n_pos] = key
            alive[n_pos] = True
            n_pos += 1
            resident.add(key)
            used += expert_bytes
            steps.append(("load", key))
        n = len(missing)
        groups.append(PlanGroup(
            layer=layer, steps=steps, prefetchable=prefetchable,
            transfer_s=n * expert_bytes / budget.bandwidth_bytes_per_s
            + budget.per_transfer_latency_s * n))
    return PlacementPlan(groups=groups, budget_bytes=budget.fast_tier_bytes,
                         expert_bytes=expert_bytes, source_fingerprint=state.fingerprint())


def apply_group_inplace(state: ResidencyState, group: PlanGroup, budget_bytes: int,
                        expert_bytes: int) -> None:
    """ref offload.py:207-222 (bookkeeping half; copies are ExpertStore's)."""
    for op, key in group.steps:
        if op == "evict":
            if key not in state.resident:
                raise ContractError(f"plan/state mismatch: evicting non-resident {key}")
            state.used_bytes -= state.resident.pop(key)
            state.fifo_order.remove(key)
        else:
            if key in state.resident:
                raise ContractError(f"plan/state mismatch: loading resident {key}")
            if state.used_bytes + expert_bytes > budget_bytes:
                raise ContractError("plan exceeds budget mid-application")
            state.resident[key] = expert_bytes
            state.fifo_order.append(key)
            state.used_bytes += expert_bytes


def apply_plan(state: ResidencyState, plan: PlacementPlan) -> tuple[ResidencyState, float]:
    """ref offload.py:225-237."""
    if plan.source_fingerprint != state.fingerprint():
        raise ContractError("plan/state mismatch: plan was computed from a different state")
    new = state.copy()
    for group in plan.groups:
        apply_group_inplace(new, group, plan.budget_bytes, plan.expert_bytes)
    new.check()
    return new, plan.estimated_transfer_s


def ensure_layer_resident(state: ResidencyState, layer: int, expert_ids, budget: MemoryBudget,
                          expert_bytes: int) -> PlanGroup:
    """Reactive single-layer load of standard serving (ref offload.py:240-278):
    evict FIFO among residents this layer does not need (the FIFO head when
    the layer's working set exceeds the budget), then load the missing
    experts in ascending order. Mutates ``state``; returns the executed group
    (bookkeeping only -- `ExpertStore` performs the copies)."""
    if expert_bytes > budget.fast_tier_bytes:
        raise UnservableError(
            f"expert of {expert_bytes} bytes exceeds budget {budget.fast_tier_bytes}")
    req = {int(e) for e in expert_ids}
    loads = [(layer, e) for e in sorted(req) if (layer, e) not in state.resident]
    steps = []
    for key in loads:
        while state.used_bytes + expert_bytes > budget.fast_tier_bytes:
            victim = next((c for c in state.fifo_order if not (c[0] == layer and c[1] in req)),
                          state.fifo_order[0])
            state.used_bytes -= state.resident.pop(victim)
            state.fifo_order.remove(victim)
            steps.append(("evict", victim))
        state.resident[key] = expert_bytes
        state.fifo_order.append(key)
        state.used_bytes += expert_bytes
        steps.append(("load", key))
    transfer_s = (len(loads) * expert_bytes / budget.bandwidth_bytes_per_s
                  + budget.per_transfer_latency_s * len(loads))
    return PlanGroup(layer=layer, steps=steps, prefetchable=False, transfer_s=transfer_s)


def effective_utilization(state: ResidencyState, activated: set) -> float:
    """ref offload.py:281-289."""
    missing = [k for k in activated if k not in state.resident]
    if missing:
        raise ContractError(f"activated experts not resident: {missing[:3]}")
    if state.used_bytes == 0:
        return 1.0
    return sum(state.resident[k] for k in activated) / state.used_bytes


def memory_reduction(table, model) -> float:
    """ref offload.py:292-300."""
    required = table.required_experts()
    return 1.0 - len(required) * model.expert_bytes_each() / model.total_expert_bytes()


# ------------------------------------------------------------------------------------
def check_device_flags(named_flags) -> None:
    """Read the kernels' device-side contract flags at a point that already
    synchronises and raise ContractError for any that is set (then clear
    them). ``named_flags``: [(what went wrong, int32 device tensor or None)].
    The flags are the grouped FFN's "routed expert without an HBM slot"
    (the tile is skipped, its rows are garbage), the permute's "expert id out
    of range" and the output projection's scatter flag."""
    flags = [(n, f) for n, f in named_flags if f is not None]
    if not flags:
        return
    vals = torch.cat([f.view(-1)[:1] for _, f in flags]).cpu().tolist()
    bad = [n for (n, _), v in zip(flags, vals) if v]
    if bad:
        for _, f in flags:
            f.zero_()
        raise ContractError("device contract check failed: " + "; ".join(sorted(set(bad))))


FFN_SLOT_MSG = "grouped FFN: a routed expert had no HBM slot (plan/slot mismatch)"
PERMUTE_MSG = "permute: expert id out of range"
OUTPROJ_MSG = "output projection: scatter contract violated"


@dataclass
class Wave:
    """Experts of one layer computed together: loads to enqueue first, then
    the FFN over ``experts`` using the expert->slot map ``slot_row``."""

    layer: int
    loads: list
    experts: list
    slot_row: np.ndarray


class RowUploader:
    """Small int32 rows (expert -> slot maps, expert lists) to the device: a
    ring of device rows written in stream order by `sida_poke_i32` (values in
    the kernel's parameter block), so they never wait behind expert copies on
    the copy engines the way a pinned H2D memcpy on the compute stream does."""

    def __init__(self, device, width: int, slots: int = 64):
        self.dev = torch.empty((slots, max(width, 1)), dtype=torch.int32, device=device)
        self.slots = slots
        self.i = 0

    def upload(self, arr: np.ndarray, stream) -> torch.Tensor:
        i = self.i
        self.i = (i + 1) % self.slots
        n = len(arr)
        src = np.ascontiguousarray(arr, dtype=np.int32)
        dst = self.dev[i, :n]
        _lib.check(_lib.lib().sida_poke_i32(dst.data_ptr(), src.ctypes.data, n, stream.cuda_stream))
        return dst


class ExpertStore:
    """HBM slot arena + pinned expert images + copy stream.

    Slots are assigned lowest-free-first; a load into a slot waits (on the copy
    stream) for the event recorded after the last FFN that read the slot.
    """


    def __init__(self, model, n_slots: int, copy_stream=None):
        if n_slots < 1:
            raise UnservableError("budget cannot hold a single expert")
        self.model = model
        self.n_slots = int(n_slots)
        self.slot_stride = model.slot_stride
        dev = model.device
        self.arena = torch.empty(self.n_slots * self.slot_stride, dtype=torch.uint8, device=dev)
        self.base_ptr = self.arena.data_ptr()
        self.err_flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.copy_stream = copy_stream or torch.cuda.Stream(device=dev)
        self.slot_of: dict = {}
        self._free = list(range(self.n_slots))
        self._reader: list = [None] * self.n_slots
        self.n_loads = 0
        self.bytes_loaded = 0
        self.peak_slots = 0
        self.rows = RowUploader(dev, model.config.num_experts)
        self.trace: list | None = None  # (name, stream, start, end) events per copy when set

    @classmethod
    def full(cls, model) -> "ExpertStore":
        """One store per model holding every expert (model_forward's default).
        It lives on the model (released with it); ``release_full(model)``
        frees its HBM arena earlier."""
        st = getattr(model, "_full_store", None)
        if st is None:
            c = model.config
            st = cls(model, c.num_layers * c.num_experts)
            model._full_store = st
        return st

    @staticmethod
    def release_full(model) -> None:
        model._full_store = None

    @classmethod
    def layer_cycling(cls, model) -> "ExpertStore":
        """A store of one layer's worth of slots (num_experts) for passes that
        visit the layers in order (the hit-rate router pass of serve_sida):
        run_layer evicts the other layers' experts before loading, so the
        arena stays at 1/L of the full one (base-128: 1.2 GB, not 14.5 GB)."""
        st = cls(model, model.config.num_experts)
        st.cycle_layers = True
        return st

    @classmethod
    def for_budget(cls, model, budget: MemoryBudget) -> "ExpertStore":
        return cls(model, budget.fast_tier_bytes // model.expert_bytes_each())

    # -- bookkeeping --------------------------------------------------------------
    def take_slot(self, key: Key) -> int:
        if key in self.slot_of:
            raise ContractError(f"plan/state mismatch: loading resident {key}")
        if not self._free:
            raise ContractError("plan exceeds budget mid-application")
        slot = heapq.heappop(self._free)
        self.slot_of[key] = slot
        self.peak_slots = max(self.peak_slots, len(self.slot_of))
        return slot

    def free_slot(self, key: Key) -> None:
        slot = self.slot_of.pop(key, None)
        if slot is None:
            raise ContractError(f"plan/state mismatch: evicting non-resident {key}")
        heapq.heappush(self._free, slot)

    def slot_row(self, layer: int, experts) -> np.ndarray:
        row = np.full(self.model.config.num_experts, -1, dtype=np.int32)
        for e in experts:
            row[e] = self.slot_of[(layer, e)]
        return row

    # -- copy engine ---------------------------------------------------------------
    def enqueue_loads(self, loads) -> torch.cuda.Event | None:
        """H2D copies for [(key, slot)], each after its slot's last reader."""
        if not loads:
            return None
        h = _lib.lib()
        cs = self.copy_stream
        for (layer, e), slot in loads:
            ev = self._reader[slot]
            if ev is not None:
                cs.wait_event(ev)
            src = self.model.expert_image(layer, e)
            if self.trace is not None:
                t0 = torch.cuda.Event(enable_timing=True)
                t0.record(cs)
            _lib.check(h.sida_expert_copy(self.base_ptr + slot * self.slot_stride, src.data_ptr(),
                                          self.slot_stride, cs.cuda_stream, None, None))
            if self.trace is not None:
                t1 = torch.cuda.Event(enable_timing=True)
                t1.record(cs)
                self.trace.append((f"copy L{layer} E{e}", "copy", t0, t1))
            self.n_loads += 1
            self.bytes_loaded += self.slot_stride
        done = torch.cuda.Event()
        done.record(cs)
        return done

    def mark_read(self, slot_row: np.ndarray, event: torch.cuda.Event) -> None:
        for s in slot_row[slot_row >= 0]:
            self._reader[int(s)] = event

    # -- one layer, every required expert resident (model_forward path) ---------------
    def run_layer(self, model, layer: int, x: torch.Tensor, dev_table, stream=None,
                  out_bf16=None, table_layer: int | None = None):
        """``table_layer``: the row of ``dev_table`` holding this layer's routing
        (default ``layer``; 0 for the single-layer tables of router mode)."""
        st = stream or torch.cuda.current_stream(model.device)
        tl = layer if table_layer is None else table_layer
        st.wait_event(dev_table.ready)
        need = [int(e) for e in np.nonzero(dev_table.hist_host()[tl])[0]]
        if getattr(self, "cycle_layers", False):
            for key in [k for k in self.slot_of if k[0] != layer]:
                self.free_slot(key)  # reuse waits on the slot's reader event
        loads = [((layer, e), self.take_slot((layer, e))) for e in need
                 if (layer, e) not in self.slot_of]
        done = self.enqueue_loads(loads)
        wave = Wave(layer, loads, need, self.slot_row(layer, need))
        return run_waves(model, [wave], x, dev_table, self, st, pre_done=[done],
                         out_bf16=out_bf16, table_layer=tl)


def run_waves(model, waves, x, dev_table, store: ExpertStore, stream, pre_done=None,
              issue=None, out_bf16=None, table_layer: int | None = None, x_perm=None,
              rows_dev=None):
    """Execute one layer as a sequence of waves on ``stream``: wait for each
    wave's copies, run the grouped FFN over its experts, record the reader
    event. ``issue(wave)`` (optional) enqueues a wave's copies just in time and
    returns their done event. ``out_bf16`` (optional) receives the layer
    output rounded to bf16 from the same epilogue. ``x_perm`` (optional) is
    the layer input already in expert-sorted bf16 rows (written by the fused
    attention output projection); without it each wave gathers. ``rows_dev``
    (optional, per wave) are device-resident expert -> slot rows: no upload,
    no reader event (the graph-replay path records those around the replay)."""
    c = model.config
    k = dev_table.k
    layer = waves[0].layer
    tables = dev_table.layer(layer if table_layer is None else table_layer)
    out = torch.empty_like(x)
    y = None
    if k > 1:
        y = torch.empty((x.shape[0] * k, c.d_model), dtype=torch.float32, device=x.device)
    multi = len(waves) > 1
    for i, wave in enumerate(waves):
        done = issue(wave) if issue is not None else (pre_done[i] if pre_done else None)
        if done is not None:
            stream.wait_event(done)
        if not wave.experts:
            continue
        row = (rows_dev[i] if rows_dev is not None
               else store.rows.upload(wave.slot_row, stream))
        elist = None
        if multi:
            elist = store.rows.upload(np.asarray(wave.experts, dtype=np.int32), stream)
        with torch.cuda.stream(stream):
            model.moe_apply_rows(tables, x, k, store, row, expert_list=elist, out=out, y=y,
                                 stream=stream, out_bf16=out_bf16, x_perm=x_perm)
        if rows_dev is None:
            ev = torch.cuda.Event()
            ev.record(stream)
            store.mark_read(wave.slot_row, ev)
    if k > 1:
        with torch.cuda.stream(stream):
            out = model.combine(y, x, k, out=out, stream=stream, out_bf16=out_bf16)
    return out
