"""Debug: fused attention core vs fp32 torch and vs the torch bf16 path, per sequence."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import _lib  # noqa: E402

lengths, d = [1, 5, 77, 128, 64, 128], 256
n = sum(lengths)
g = torch.Generator(device="cuda")
g.manual_seed(n + d)
qkv = (torch.randn((n, 3 * d), generator=g, device="cuda") * 0.5).to(torch.bfloat16)
off = np.zeros(len(lengths) + 1, dtype=np.int32)
np.cumsum(lengths, out=off[1:])
seq_off = torch.from_numpy(off).cuda()
ctx = torch.full((n, d), float("nan"), dtype=torch.bfloat16, device="cuda")
_lib.check(_lib.lib().sida_attention_core(qkv.data_ptr(), seq_off.data_ptr(), len(lengths), n,
                                          max(lengths), d, ctx.data_ptr(), None))
torch.cuda.synchronize()
q, k, v = qkv.float().split(d, dim=1)
qb, kb, vb = qkv.split(d, dim=1)
for s in range(len(lengths)):
    a, b = int(off[s]), int(off[s + 1])
    att = torch.softmax(q[a:b] @ k[a:b].T / d ** 0.5, dim=-1)
    ref = att @ v[a:b]
    sc = torch.mm(qb[a:b], kb[a:b].T, out_dtype=torch.float32) / d ** 0.5
    tb = torch.softmax(sc, dim=-1).to(torch.bfloat16) @ vb[a:b]
    rms = ref.pow(2).mean().sqrt().item()
    e1 = (ctx[a:b].float() - ref).abs().max().item() / rms
    e2 = (tb.float() - ref).abs().max().item() / rms
    print(f"T={b - a}: fused max err {e1:.3e} rms, torch-bf16 path {e2:.3e} rms, rms {rms:.3f}, "
          f"max|att| {att.max().item():.3f}")
