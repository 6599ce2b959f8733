"""cProfile of the host side of the serving loop at a small batch (where the
host, not the GPU, bounds the step): python tools/host_profile.py --experts 256"""
import argparse
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MemoryBudget, MoEConfig, MoEModel, PredictorConfig  # noqa: E402
from paper_2310_18859_b200 import PredictorNet, Rng  # noqa: E402
from paper_2310_18859_b200.engine import SidaEngine  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--experts", type=int, default=256)
p.add_argument("--batch", type=int, default=1)
p.add_argument("--seq", type=int, default=128)
p.add_argument("--steps", type=int, default=20)
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts,
                expert_hidden=3072, max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
eng = SidaEngine(model, pred, MemoryBudget(model.total_expert_bytes()))
n = a.batch * a.seq
lengths = [a.seq] * a.batch
toks = [torch.randint(0, cfg.vocab_size, (n,), device="cuda", dtype=torch.int32)
        for _ in range(a.steps + 5)]


def run(k0, k1):
    tabs = {k0: eng.hash_tokens(k0, toks[k0], lengths)}
    for j in range(k0, k1):
        tabs[j + 1] = eng.hash_tokens(j + 1, toks[j + 1], lengths)
        eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j], next_table=tabs[j + 1])
    torch.cuda.synchronize()


run(0, 3)
pr = cProfile.Profile()
pr.enable()
run(3, 3 + a.steps)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(25)
