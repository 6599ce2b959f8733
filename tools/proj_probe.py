"""Time sida_out_proj_scatter alone at the bench shape (N=32768, d=768, k=1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import _lib  # noqa: E402

n, d, k = 32768, 768, 1
h = _lib.lib()
ctx = torch.randn((n, d), device="cuda").to(torch.bfloat16)
wo_t = torch.zeros(h.sida_out_proj_bytes(d) // 2, dtype=torch.bfloat16, device="cuda")
wo_t[: d * d] = (torch.randn(d * d, device="cuda") / d ** 0.5).to(torch.bfloat16)
resid = torch.randn((n, d), device="cuda")
out = torch.empty_like(resid)
inv = torch.randperm(n, device="cuda").to(torch.int32)
xp = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def run():
    _lib.check(h.sida_out_proj_scatter(ctx.data_ptr(), n, d, wo_t.data_ptr(), resid.data_ptr(),
                                       out.data_ptr(), inv.data_ptr(), k, xp.data_ptr(),
                                       err.data_ptr(), st))


for _ in range(3):
    run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
byts = n * d * (2 + 4 + 4 + 2)
print(f"out_proj_scatter: {ms * 1e3:.1f} us, {2 * n * d * d / ms / 1e9:.0f} TFLOP/s, "
      f"{byts / ms / 1e6:.0f} GB/s of algorithmic bytes")
