"""How much does the hash stream (batch j+1) slow the forward (batch j)?

Times K forwards (a) with every table built beforehand and (b) pipelined the
way bench.py runs them, and (c) the hash alone.

    python tools/overlap_probe.py [--steps 10]
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
p.add_argument("--steps", type=int, default=10)
p.add_argument("--batch", type=int, default=256)
p.add_argument("--seq", type=int, default=128)
p.add_argument("--experts", type=int, default=8)
a = p.parse_args()
cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=a.experts, expert_hidden=3072,
                max_seq_len=512)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, a.experts, Rng(1))
eng = SidaEngine(model, pred, MemoryBudget(model.total_expert_bytes()))
n = a.batch * a.seq
lengths = [a.seq] * a.batch
toks = [torch.randint(0, cfg.vocab_size, (n,), device="cuda", dtype=torch.int32)
        for _ in range(a.steps + 4)]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
cs = eng.compute_stream

# warm-up
tabs = {0: eng.hash_tokens(0, toks[0], lengths)}
for j in range(3):
    tabs[j + 1] = eng.hash_tokens(j + 1, toks[j + 1], lengths)
    eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j])
torch.cuda.synchronize()

# (c) hash alone
e0, e1 = ev(), ev()
e0.record(eng.hash_stream)
pre = [eng.hash_tokens(j, toks[j], lengths) for j in range(a.steps)]
e1.record(eng.hash_stream)
torch.cuda.synchronize()
hash_ms = e0.elapsed_time(e1) / a.steps

# (a) forwards only
e0, e1 = ev(), ev()
e0.record(cs)
for j in range(a.steps):
    eng.forward(pre[j], lengths, tokens_dev=toks[j])
e1.record(cs)
torch.cuda.synchronize()
fwd_ms = e0.elapsed_time(e1) / a.steps

# (b) pipelined
tabs = {0: eng.hash_tokens(0, toks[0], lengths)}
torch.cuda.synchronize()
e0, e1 = ev(), ev()
e0.record(cs)
for j in range(a.steps):
    tabs[j + 1] = eng.hash_tokens(j + 1, toks[j + 1], lengths)
    eng.forward(tabs.pop(j), lengths, tokens_dev=toks[j])
e1.record(cs)
torch.cuda.synchronize()
pipe_ms = e0.elapsed_time(e1) / a.steps
print(f"hash alone {hash_ms:.3f} ms, forward alone {fwd_ms:.3f} ms, pipelined {pipe_ms:.3f} ms "
      f"per step ({n} tokens): interference {pipe_ms - fwd_ms:.3f} ms")
