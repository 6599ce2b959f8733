"""End-to-end serve_sida timing at the bench shape (host batches in, host
logits out), repeated, with a host profile of one call: where does the e2e
wall clock go?   python tools/e2e_probe.py [--experts 128] [--reps 4]"""
import argparse
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MemoryBudget, MoEConfig, MoEModel  # noqa: E402
from paper_2310_18859_b200 import PredictorConfig, PredictorNet, Rng, SequenceBatch  # noqa: E402
from paper_2310_18859_b200 import serve_sida  # noqa: E402
from paper_2310_18859_b200.engine import SidaEngine  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--experts", type=int, default=128)
p.add_argument("--batches", type=int, default=10)
p.add_argument("--reps", type=int, default=4)
p.add_argument("--budget-frac", type=float, default=0.97)
p.add_argument("--victim-policy", default="fifo", choices=["fifo", "spread"])
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=3072, max_seq_len=512, num_classes=2)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
eb = model.expert_bytes_each()
slots = int(round(a.budget_frac * 12 * a.experts))
budget = MemoryBudget(slots * eb)
eng = SidaEngine(model, pred, budget, victim_policy=a.victim_policy)
rng = np.random.default_rng(99)
B, T = 256, 128


def batches(n, i0):
    return [SequenceBatch(i0 + i, [rng.integers(0, cfg.vocab_size, size=T) for _ in range(B)])
            for i in range(n)]


serve_sida(model, pred, batches(3, 0), budget, engine=eng, compute_hit_rate=False)
for r in range(a.reps):
    bs = batches(a.batches, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = serve_sida(model, pred, bs, budget, engine=eng, compute_hit_rate=False)
    dt = time.perf_counter() - t0
    lat = [b["latency_s"] * 1e3 for b in rep.batch_records]
    print(f"rep {r}: {dt * 1e3:.1f} ms wall for {a.batches} batches = "
          f"{a.batches * B * T / dt / 1e6:.3f} M tok/s; device latency per batch "
          f"{np.round(lat, 2).tolist()}")
bs = batches(a.batches, 0)
torch.cuda.synchronize()
prof = cProfile.Profile()
prof.enable()
serve_sida(model, pred, bs, budget, engine=eng, compute_hit_rate=False)
prof.disable()
pstats.Stats(prof).sort_stats("tottime").print_stats(15)
pstats.Stats(prof).sort_stats("cumulative").print_stats(25)
