"""sida_permute_hist over L layers (+ one layer's bf16 row gather) for ncu.

    python tools/permute_probe.py [--layers 12] [--rows 262144] [--experts 256] [--iters 3]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import _lib  # noqa: E402
from paper_2310_18859_b200.predictor import DeviceTable  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--layers", type=int, default=12)
p.add_argument("--rows", type=int, default=262144)
p.add_argument("--experts", type=int, default=256)
p.add_argument("--d", type=int, default=768)
p.add_argument("--iters", type=int, default=3)
a = p.parse_args()
L, N, K = a.layers, a.rows, a.experts
ids = torch.randint(0, K, (L, N, 1), device="cuda", dtype=torch.int32)
al = torch.rand((L, N, 1), device="cuda", dtype=torch.float64)
dt = DeviceTable(ids, al, al.float(), N, 1)
x = torch.randn(N, a.d, device="cuda")
xp = torch.empty((N, a.d), dtype=torch.bfloat16, device="cuda")
st = torch.cuda.current_stream()
for _ in range(a.iters):
    dt.permute(K, st)
    _lib.check(_lib.lib().sida_gather_rows_bf16(x.data_ptr(), dt.perm[0].data_ptr(), N, 1, a.d,
                                                xp.data_ptr(), st.cuda_stream))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record(st)
for _ in range(reps):
    dt.permute(K, st)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
# SURVEY §8(d) algorithmic bytes: ids + perm + inv (4 B each per row) + 8 K, plus the
# alpha row read and alpha_perm write of this path (4 B each)
byts = L * (N * (4 + 4 + 4 + 4 + 4) + 8 * K)
print(f"permute L={L} rows={N} K={K}: {ms * 1e3:.1f} us per call, {byts / ms / 1e6:.0f} GB/s "
      f"({byts / 1e6:.1f} MB)")
