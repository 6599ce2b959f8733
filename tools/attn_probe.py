"""Time attention_mix alone (back to back on one stream) at the bench shape,
and the host enqueue rate of one full forward, to separate GPU time from
launch gaps.

    python tools/attn_probe.py [--batch 256] [--seq 128]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MoEConfig, MoEModel  # noqa: E402
from paper_2310_18859_b200.moe import BatchLayout  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=256)
p.add_argument("--seq", type=int, default=128)
p.add_argument("--iters", type=int, default=24)
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=2, num_experts=8, expert_hidden=3072,
                max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
n = a.batch * a.seq
toks = torch.randint(0, cfg.vocab_size, (n,), device="cuda", dtype=torch.int32)
lay = BatchLayout([a.seq] * a.batch, toks, model.device)
x = model.embed_layout(lay)
xb = x.to(torch.bfloat16)
for _ in range(3):
    model.attention_mix(0, x, lay, xb=xb)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(a.iters):
    model.attention_mix(0, x, lay, xb=xb)
e1.record()
t_host = time.perf_counter() - t0
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
d = cfg.d_model
fl = 2 * n * d * 3 * d + 2 * n * a.seq * d * 2 + 2 * n * d * d
print(f"attention_mix: {ms:.3f} ms/layer on the GPU, host enqueue {t_host / a.iters * 1e3:.3f} "
      f"ms/layer, {fl / ms / 1e9:.1f} TFLOP/s (N={n}, T={a.seq})")
