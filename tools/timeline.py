"""Copy / compute / hash overlap timeline of SiDA serving (the evidence the
missing nsys would give): CUDA events on the hash, compute and copy streams
around every hash, attention, FFN and expert copy of a few serving steps,
written as a chrome://tracing JSON plus an overlap summary.

    python tools/timeline.py [--experts 128] [--budget-frac 0.97] [--out gpurun_out/timeline.json]

exposed copy time = copy busy time not covered by any compute-stream span.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MemoryBudget, MoEConfig, MoEModel  # noqa: E402
from paper_2310_18859_b200 import PredictorConfig, PredictorNet, Rng  # noqa: E402
from paper_2310_18859_b200.engine import SidaEngine  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--experts", type=int, default=128)
p.add_argument("--budget-frac", type=float, default=0.97)
p.add_argument("--policy", default="spread")
p.add_argument("--batch", type=int, default=256)
p.add_argument("--seq", type=int, default=128)
p.add_argument("--steps", type=int, default=3)
p.add_argument("--warmup", type=int, default=3)
p.add_argument("--out", default="gpurun_out/timeline.json")
a = p.parse_args()

cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=3072, max_seq_len=512, num_classes=2)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
eb = model.expert_bytes_each()
slots = int(round(a.budget_frac * cfg.num_layers * cfg.num_experts))
eng = SidaEngine(model, pred, MemoryBudget(slots * eb), victim_policy=a.policy)
n = a.batch * a.seq
lengths = [a.seq] * a.batch
g = torch.Generator(device="cuda")
g.manual_seed(5)
toks = [torch.randint(0, cfg.vocab_size, (n,), device="cuda", dtype=torch.int32, generator=g)
        for _ in range(a.warmup + a.steps + 1)]
tabs = {0: eng.hash_tokens(0, toks[0], lengths)}
base = torch.cuda.Event(enable_timing=True)
for j in range(a.warmup + a.steps):
    if j == a.warmup:
        torch.cuda.synchronize()
        base.record(eng.compute_stream)
        eng.trace, eng.store.trace = [], []
    tabs[j + 1] = eng.hash_tokens(j + 1, toks[j + 1], lengths)
    eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j], next_table=tabs[j + 1])
torch.cuda.synchronize()
spans = []
for name, stream, e0, e1 in eng.trace + eng.store.trace:
    spans.append((stream, name, base.elapsed_time(e0), base.elapsed_time(e1)))
trace = {"traceEvents": [{"name": nm, "ph": "X", "ts": t0 * 1e3, "dur": (t1 - t0) * 1e3,
                          "pid": 0, "tid": st} for st, nm, t0, t1 in spans],
         "displayTimeUnit": "ms"}


def union(iv):
    iv = sorted(iv)
    out = []
    for s, e in iv:
        if out and s <= out[-1][1]:
            out[-1][1] = max(out[-1][1], e)
        else:
            out.append([s, e])
    return out


comp = union([(t0, t1) for st, _, t0, t1 in spans if st == "compute"])
copy = union([(t0, t1) for st, _, t0, t1 in spans if st == "copy"])
copy_ms = sum(e - s for s, e in copy)
covered = 0.0
for s, e in copy:
    for cs, ce in comp:
        covered += max(0.0, min(e, ce) - max(s, cs))
total = max(t1 for _, _, _, t1 in spans)
summary = {"experts": a.experts, "budget_frac": a.budget_frac, "policy": a.policy, "steps": a.steps,
           "ms_per_step": total / a.steps, "copies": sum(1 for s in spans if s[0] == "copy"),
           "copy_busy_ms": copy_ms, "copy_overlapped_with_compute_ms": covered,
           "copy_exposed_ms": copy_ms - covered,
           "hash_busy_ms": sum(t1 - t0 for st, _, t0, t1 in spans if st == "hash")}
trace["summary"] = summary
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
json.dump(trace, open(a.out, "w"))
print(json.dumps(summary))
