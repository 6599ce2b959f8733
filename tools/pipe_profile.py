"""Pipelined serving loop (as tools/sweep.py) at chosen shapes: per-step
device times, then one profiled step's CUDA runtime calls (host stalls:
cudaMalloc, synchronizes) and top kernels.

    python tools/pipe_profile.py --shapes 64x256,1x128
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MemoryBudget, MoEConfig, MoEModel, PredictorConfig  # noqa: E402
from paper_2310_18859_b200 import PredictorNet, Rng  # noqa: E402
from paper_2310_18859_b200.engine import SidaEngine  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--shapes", default="64x256,1x128")
p.add_argument("--experts", type=int, default=8)
p.add_argument("--steps", type=int, default=8)
p.add_argument("--profile-first", action="store_true",
               help="profile the first steps of each shape (first-use stalls)")
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=3072, max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
eng = SidaEngine(model, pred, MemoryBudget(model.total_expert_bytes()))
cs = eng.compute_stream
for shp in a.shapes.split(","):
    B, T = (int(v) for v in shp.split("x"))
    lengths = [T] * B
    toks = [torch.randint(0, cfg.vocab_size, (B * T,), device="cuda", dtype=torch.int32)
            for _ in range(a.steps + 4)]
    from torch.profiler import ProfilerActivity, profile
    prof0 = profile(activities=[ProfilerActivity.CPU]) if a.profile_first else None
    if prof0:
        prof0.__enter__()
    tabs = {0: eng.hash_tokens(0, toks[0], lengths)}
    times = []
    for j in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        tabs[j + 1] = eng.hash_tokens(j + 1, toks[j + 1], lengths)
        eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j], next_table=tabs[j + 1])
        e1.record(cs)
        times.append((e0, e1))
    torch.cuda.synchronize()
    if prof0:
        prof0.__exit__(None, None, None)
        ev = sorted(prof0.key_averages(), key=lambda e: -e.self_cpu_time_total)
        for e in ev[:15]:
            print(f"  first-steps host {e.key[:50]:50s} calls {e.count:5d} "
                  f"self {e.self_cpu_time_total / 1e3:.3f} ms")
    print(f"B={B} T={T} step ms:", [round(x.elapsed_time(y), 3) for x, y in times], flush=True)
    from torch.profiler import ProfilerActivity, profile
    j = a.steps
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for i in range(2):
            tabs[j + 1] = eng.hash_tokens(j + 1, toks[j + 1], lengths)
            eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j], next_table=tabs[j + 1])
            j += 1
        torch.cuda.synchronize()
    ka = prof.key_averages()
    rt = [e for e in ka if e.key.startswith("cuda") or "Synchronize" in e.key or "Malloc" in e.key]
    rt.sort(key=lambda e: -e.cpu_time_total)
    for e in rt[:10]:
        print(f"  host {e.key:40s} calls {e.count:5d} total {e.cpu_time_total / 1e3:.3f} ms")
    ks = [e for e in ka if e.device_time_total > 0]
    ks.sort(key=lambda e: -e.device_time_total)
    for e in ks[:10]:
        print(f"  dev  {e.key[:60]:60s} calls {e.count:5d} total {e.device_time_total / 1e3:.3f} ms")
    print(f"  python-side CPU total (2 steps) "
          f"{sum(e.self_cpu_time_total for e in ka) / 1e3:.3f} ms", flush=True)
    del toks, tabs
