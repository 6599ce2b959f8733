"""A/B of the hash/compute stream arrangement at the bench shape, in one
process, modes interleaved and repeated (median ms per step):
  prio    hash stream at low priority, compute at high
  hashprio  hash stream at high priority, compute at low
  flat    both streams at the same priority
  serial  hash enqueued on the compute stream (no overlap)
    python tools/pipe_ab.py [--experts 128] [--reps 5] [--steps 8]
"""
import argparse
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
p.add_argument("--batch", type=int, default=256)
p.add_argument("--seq", type=int, default=128)
p.add_argument("--steps", type=int, default=8)
p.add_argument("--reps", type=int, default=5)
p.add_argument("--ahead", type=int, default=2)
p.add_argument("--modes", default="prio,flat,serial")
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=3072, max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
budget = MemoryBudget(model.total_expert_bytes())
lo, hi = torch.cuda.Stream.priority_range()
cs_hi = torch.cuda.Stream(priority=hi)
streams = {"prio": (torch.cuda.Stream(priority=lo), cs_hi),
           "hashprio": (torch.cuda.Stream(priority=hi), torch.cuda.Stream(priority=lo)),
           "flat": (torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=0)),
           "serial": (cs_hi, cs_hi)}
modes = a.modes.split(",")
engines = {}
store = None
for m in modes:
    engines[m] = SidaEngine(model, pred, budget, streams=streams[m], store=store)
    store = engines[m].store
n = a.batch * a.seq
lengths = [a.seq] * a.batch
toks = [torch.randint(0, cfg.vocab_size, (n,), device="cuda", dtype=torch.int32)
        for _ in range(a.steps + a.ahead + 4)]


def run(eng, steps):
    A = a.ahead
    tabs = {i: eng.hash_tokens(i, toks[i], lengths) for i in range(A)}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for j in range(steps + 2):
        if j == 2:
            e0.record(eng.compute_stream)
        tabs[j + A] = eng.hash_tokens(j + A, toks[(j + A) % len(toks)], lengths)
        eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j], next_table=tabs[j + 1])
    e1.record(eng.compute_stream)
    torch.cuda.synchronize()
    for t in tabs.values():
        pass
    return e0.elapsed_time(e1) / steps


for m in modes:
    run(engines[m], 2)
res = {m: [] for m in modes}
for r in range(a.reps):
    for m in modes:
        res[m].append(run(engines[m], a.steps))
for m in modes:
    v = np.array(res[m])
    print(f"{m:7s} median {np.median(v):.3f} ms/step  (min {v.min():.3f}, max {v.max():.3f})")
