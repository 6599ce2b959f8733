"""Repeat one serving point R times in one process (device step times) to
expose bimodal step times.  python tools/variance_probe.py --experts 256 --batch 256 --seq 128"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MemoryBudget, MoEConfig, MoEModel, PredictorConfig  # noqa: E402
from paper_2310_18859_b200 import PredictorNet, Rng  # noqa: E402
from paper_2310_18859_b200.engine import SidaEngine  # noqa: E402
from paper_2310_18859_b200.predictor import ExpertHashTable  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--experts", type=int, default=256)
p.add_argument("--batch", type=int, default=256)
p.add_argument("--seq", type=int, default=128)
p.add_argument("--steps", type=int, default=5)
p.add_argument("--reps", type=int, default=8)
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=3072, max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
eng = SidaEngine(model, pred, MemoryBudget(model.total_expert_bytes()))
wl = [128] * 64
wt = torch.randint(0, cfg.vocab_size, (sum(wl),), device="cuda", dtype=torch.int32)
ids = np.tile(np.arange(sum(wl)) % a.experts, (12, 1))[:, :, None]
eng.forward(ExpertHashTable(0, wl, ids, np.ones(ids.shape)), wl, tokens_dev=wt)
torch.cuda.synchronize()
n = a.batch * a.seq
lengths = [a.seq] * a.batch
toks = [torch.randint(0, cfg.vocab_size, (n,), device="cuda", dtype=torch.int32)
        for _ in range(a.steps + 4)]
bid = 1
res = []
for r in range(a.reps):
    tabs = {0: eng.hash_tokens(bid, toks[0], lengths)}
    bid += 1
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for j in range(a.steps + 2):
        if j == 2:
            torch.cuda.synchronize()
            e0.record(eng.compute_stream)
        tabs[j + 1] = eng.hash_tokens(bid, toks[(j + 1) % len(toks)], lengths)
        bid += 1
        eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j % len(toks)], next_table=tabs[j + 1])
    e1.record(eng.compute_stream)
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / a.steps)
print("ms/step per rep:", " ".join(f"{v:.2f}" for v in res))
