"""Per-call hash timing across batch shapes, with a kernel breakdown (torch
profiler / CUPTI) for each: python tools/hash_shapes.py --shapes 1x128,8x128"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MoEConfig, MoEModel, PredictorConfig, PredictorNet, Rng  # noqa
from paper_2310_18859_b200.predictor import hash_device  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--shapes", default="1x128,8x128,64x128,256x128,8x256,64x256,64x512")
p.add_argument("--experts", type=int, default=8)
p.add_argument("--iters", type=int, default=6)
p.add_argument("--profile", action="store_true")
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=64, max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
st = torch.cuda.Stream()
for shp in a.shapes.split(","):
    B, T = (int(v) for v in shp.split("x"))
    lengths = [T] * B
    toks = torch.randint(0, cfg.vocab_size, (B * T,), device="cuda", dtype=torch.int32)
    for _ in range(2):
        hash_device(pred, model, toks, lengths, 1, 0, st)
    torch.cuda.synchronize()
    dev, host = [], []
    for i in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        t0 = time.perf_counter()
        hash_device(pred, model, toks, lengths, 1, i, st)
        host.append((time.perf_counter() - t0) * 1e3)
        e1.record(st)
        torch.cuda.synchronize()
        dev.append(e0.elapsed_time(e1))
    print(f"B={B} T={T}: device ms {[round(x, 3) for x in dev]} host ms "
          f"{[round(x, 3) for x in host]}", flush=True)
    if a.profile:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            hash_device(pred, model, toks, lengths, 1, 0, st)
            torch.cuda.synchronize()
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12), flush=True)
