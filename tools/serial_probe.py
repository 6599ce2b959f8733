"""GPU-side timeline of serve_sida with the hash on the compute stream
(SIDA_HASH_SERIAL=1): CUDA events around every hash+permute (ring.produce) and
every forward, plus the host time spent inside each call, to locate the idle
gaps between them.   SIDA_HASH_SERIAL=1 python tools/serial_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MemoryBudget, MoEConfig, MoEModel  # noqa: E402
from paper_2310_18859_b200 import PredictorConfig, PredictorNet, Rng, SequenceBatch  # noqa: E402
from paper_2310_18859_b200 import serve_sida  # noqa: E402
from paper_2310_18859_b200.engine import SidaEngine  # noqa: E402
from paper_2310_18859_b200.predictor import DeviceTableRing  # noqa: E402

cfg = MoEConfig(vocab_size=32128, d_model=768, num_layers=12, num_experts=128,
                expert_hidden=3072, max_seq_len=512, num_classes=2)
model = MoEModel.synthetic(cfg, 0)
pred = PredictorNet(PredictorConfig(), 768, 12, 128, Rng(1))
eb = model.expert_bytes_each()
budget = MemoryBudget(int(round(0.97 * 12 * 128)) * eb)
eng = SidaEngine(model, pred, budget, victim_policy="fifo")
rng = np.random.default_rng(99)
B, T = 256, 128
spans = []  # (name, ev0, ev1, host_s)


def batches(n):
    return [SequenceBatch(i, [rng.integers(0, cfg.vocab_size, size=T) for _ in range(B)])
            for i in range(n)]


orig_fwd, orig_prod = SidaEngine.forward, DeviceTableRing.produce


def fwd(self, table, *a, **k):
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(self.compute_stream)
    h0 = time.perf_counter()
    out = orig_fwd(self, table, *a, **k)
    h1 = time.perf_counter()
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(self.compute_stream)
    spans.append((f"fwd {table.batch_id}", e0, e1, h0, h1))
    return out


def prod(self, predictor, model_, lengths, k, stream, batch_id, **kw):
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h0 = time.perf_counter()
    out = orig_prod(self, predictor, model_, lengths, k, stream, batch_id, **kw)
    h1 = time.perf_counter()
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(stream)
    spans.append((f"hash {batch_id}", e0, e1, h0, h1))
    return out


serve_sida(model, pred, batches(3), budget, engine=eng, compute_hit_rate=False)
SidaEngine.forward, DeviceTableRing.produce = fwd, prod
bs = batches(12)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
h00 = time.perf_counter()
rep = serve_sida(model, pred, bs, budget, engine=eng, compute_hit_rate=False)
torch.cuda.synchronize()
print(f"wall {rep.total_wall_s * 1e3:.1f} ms for {len(bs)} batches")
rows = sorted(((t0.elapsed_time(e0), t0.elapsed_time(e1), n, (h0 - h00) * 1e3, (h1 - h00) * 1e3)
               for n, e0, e1, h0, h1 in spans))
prev = None
for g0, g1, n, h0, h1 in rows:
    gap = g0 - prev if prev is not None else 0.0
    print(f"{n:10s} gpu {g0:8.2f} -> {g1:8.2f} ({g1 - g0:6.2f} ms, gap before {gap:5.2f})  "
          f"host call {h0:8.2f} -> {h1:8.2f} ({h1 - h0:5.2f} ms)")
    prev = g1
