"""Time the fp64 hash (+permute) at the bench shape: python tools/hash_probe.py"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MoEConfig, MoEModel, PredictorConfig, PredictorNet, Rng  # noqa
from paper_2310_18859_b200.predictor import hash_device  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=256)
p.add_argument("--seq", type=int, default=128)
p.add_argument("--experts", type=int, default=8)
p.add_argument("--layers", type=int, default=12)
p.add_argument("--iters", type=int, default=10)
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=a.layers, num_experts=a.experts,
                expert_hidden=64, max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, a.layers, a.experts, Rng(1))
n = a.batch * a.seq
toks = torch.randint(0, cfg.vocab_size, (n,), device="cuda", dtype=torch.int32)
st = torch.cuda.current_stream()
lengths = [a.seq] * a.batch
for _ in range(2):
    hash_device(pred, model, toks, lengths, 1, 0, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(a.iters):
    hash_device(pred, model, toks, lengths, 1, i, st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(f"hash+permute: {ms:.3f} ms per batch of {n} tokens ({n / ms / 1e3:.1f} M tok/s)")
if os.environ.get("SIDA_HASH_PROF"):
    import numpy as np
    from paper_2310_18859_b200 import _lib
    out = np.zeros(6, dtype=np.uint64)
    _lib.check(_lib.load().sida_debug_hash_prof(out.ctypes.data))
    names = ["scores", "sort", "support", "ctx", "heads", "setup"]
    tot = float(out.sum())
    print("attn phases: " + ", ".join(f"{n} {v / tot:.1%}" for n, v in zip(names, out)))
