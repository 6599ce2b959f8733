"""Host time per serving step at the bench shape vs the device step time: is
the launch loop ahead of the GPU?  python tools/host_time.py [--budget-frac 0.9]"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MemoryBudget, MoEConfig, MoEModel, PredictorConfig  # noqa: E402
from paper_2310_18859_b200 import PredictorNet, Rng  # noqa: E402
from paper_2310_18859_b200.engine import SidaEngine  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--experts", type=int, default=8)
p.add_argument("--batch", type=int, default=256)
p.add_argument("--seq", type=int, default=128)
p.add_argument("--steps", type=int, default=10)
p.add_argument("--budget-frac", type=float, default=0.9)
p.add_argument("--victim-policy", default="spread")
p.add_argument("--ahead", type=int, default=2, help="batches hashed ahead of the forward")
p.add_argument("--profile", action="store_true", help="cProfile the timed forwards")
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=3072, max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
slots = int(round(a.budget_frac * 12 * a.experts))
eng = SidaEngine(model, pred, MemoryBudget(slots * model.expert_bytes_each()),
                 victim_policy=a.victim_policy)
n = a.batch * a.seq
lengths = [a.seq] * a.batch
toks = [torch.randint(0, cfg.vocab_size, (n,), device="cuda", dtype=torch.int32)
        for _ in range(a.steps + 5)]
A = a.ahead
tabs = {i: eng.hash_tokens(i, toks[i], lengths) for i in range(A)}
for j in range(3):
    tabs[j + A] = eng.hash_tokens(j + A, toks[j + A], lengths)
    eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j], next_table=tabs[j + 1])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
host = []
if a.profile:
    import cProfile
    prof = cProfile.Profile()
    prof.enable()
e0.record(eng.compute_stream)
for j in range(3, 3 + a.steps):
    t0 = time.perf_counter()
    tabs[j + A] = eng.hash_tokens(j + A, toks[(j + A) % len(toks)], lengths)
    t1 = time.perf_counter()
    eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j], next_table=tabs[j + 1])
    host.append((t1 - t0, time.perf_counter() - t1))
e1.record(eng.compute_stream)
t_end = time.perf_counter()
torch.cuda.synchronize()
dev = e0.elapsed_time(e1) / a.steps
hh = sum(h for h, _ in host) / len(host) * 1e3
ff = sum(f for _, f in host) / len(host) * 1e3
if a.profile:
    import pstats
    prof.disable()
    pstats.Stats(prof).sort_stats("tottime").print_stats(18)
print(f"host per step: hash {hh:.2f} ms + forward {ff:.2f} ms = {hh + ff:.2f} ms; "
      f"device step {dev:.2f} ms")
