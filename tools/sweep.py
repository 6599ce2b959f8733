"""Serving sweep over batch size and sequence length (BASELINE configs[4] grid,
on one B200): tokens/s of the device-resident pipeline (hash one batch ahead,
all experts resident) per (batch, seq), for a Switch-base shape.

    python tools/sweep.py --experts 256 --batches 1,8,64,256,512 --seqs 128,256,512

Prints one JSON line per point and writes the table to --out (JSON).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MemoryBudget, MoEConfig, MoEModel, PredictorConfig  # noqa: E402
from paper_2310_18859_b200 import PredictorNet, Rng  # noqa: E402
from paper_2310_18859_b200.engine import SidaEngine  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--experts", type=int, default=256)
p.add_argument("--batches", default="1,8,64,256,512")
p.add_argument("--seqs", default="128,256,512")
p.add_argument("--steps", type=int, default=5)
p.add_argument("--warmup", type=int, default=3)
p.add_argument("--max-tokens", type=int, default=131072)
p.add_argument("--out", default="")
a = p.parse_args()

cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=3072, max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
eng = SidaEngine(model, pred, MemoryBudget(model.total_expert_bytes()))
# warm the expert store: a forward whose table routes token t to expert
# t % K in every layer makes every expert of every layer resident, so no point
# of the sweep pays first-touch expert copies (the predictor's skewed routing
# alone can leave rarely used experts cold until some later point)
from paper_2310_18859_b200.predictor import ExpertHashTable  # noqa: E402

wl = [128] * 64
wt = torch.randint(0, cfg.vocab_size, (sum(wl),), device="cuda", dtype=torch.int32)
ids = np.tile(np.arange(sum(wl)) % a.experts, (12, 1))[:, :, None]
eng.forward(ExpertHashTable(0, wl, ids, np.ones(ids.shape)), wl, tokens_dev=wt)
for i in range(2):
    eng.forward(eng.hash_tokens(i + 1, wt, wl), wl, tokens_dev=wt)
torch.cuda.synchronize()
rows = []
for T in [int(v) for v in a.seqs.split(",")]:
    for B in [int(v) for v in a.batches.split(",")]:
        n = B * T
        if n > a.max_tokens:
            continue
        lengths = [T] * B
        g = torch.Generator(device="cuda")
        g.manual_seed(B * 1000 + T)
        toks = [torch.randint(0, cfg.vocab_size, (n,), generator=g, device="cuda",
                              dtype=torch.int32) for _ in range(a.steps + a.warmup + 1)]
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
        tabs = {0: eng.hash_tokens(0, toks[0], lengths)}
        for j in range(a.steps + a.warmup):
            if j == a.warmup:
                torch.cuda.synchronize()
                evs[0].record(eng.compute_stream)
            tabs[j + 1] = eng.hash_tokens(j + 1, toks[j + 1], lengths)
            eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j], next_table=tabs[j + 1])
            if j >= a.warmup:
                evs[j - a.warmup + 1].record(eng.compute_stream)
        torch.cuda.synchronize()
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(a.steps)]
        ms = evs[0].elapsed_time(evs[-1]) / a.steps
        med = float(np.median(per))
        # the median step is reported beside the mean: a one-off stall inside
        # the timed steps (seen sporadically when the shape changes between
        # points) moves the mean, not the median
        row = {"experts": a.experts, "batch": B, "seq": T, "tokens_per_step": n,
               "ms_per_step": ms, "tokens_per_s": n / (ms / 1e3),
               "median_ms_per_step": med, "max_ms_step": max(per),
               "tokens_per_s_median": n / (med / 1e3)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del toks, tabs
        torch.cuda.empty_cache()
if a.out:
    json.dump({"workload": f"Switch-base-{a.experts} shape (d=768, h=3072, 12 layers), bf16, "
                           "all experts resident, synthetic uniform tokens, 1 B200",
               "points": rows}, open(a.out, "w"), indent=1)
