"""Forward-only step time at the bench shape (tables hashed beforehand, no
hash/compute overlap, every expert resident): eager launches vs CUDA-graph
replay, to separate launch/host overhead from kernel time.

    python tools/fwd_probe.py [--experts 128] [--steps 8]
"""
import argparse
import os
import sys

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
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=3072, max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
eng = SidaEngine(model, pred, MemoryBudget(model.total_expert_bytes()))
n = a.batch * a.seq
lengths = [a.seq] * a.batch
tok = torch.randint(0, cfg.vocab_size, (n,), device="cuda", dtype=torch.int32)


def run(steps, graph):
    eng.graph_max_tokens = n if graph else 0
    tabs = [eng.hash_tokens(i, tok, lengths) for i in range(2)]
    torch.cuda.synchronize()
    cs = eng.compute_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for j in range(steps + 3):
        if j == 3:
            e0.record(cs)
        eng.forward(tabs[j % 2], lengths, tokens_dev=tok)
    e1.record(cs)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for g in (False, True, False, True):
    ms = run(a.steps, g)
    print(f"{'graph' if g else 'eager'}: {ms:.3f} ms/step forward only "
          f"({n / ms / 1e3:.2f} M tok/s), graph replays {eng.graph_replays}")
