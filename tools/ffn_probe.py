"""Run one MoE layer's grouped FFN at the bench shape (for ncu / timing).

    python tools/ffn_probe.py [--tokens 32768] [--experts 8] [--iters 20]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_18859_b200 import MoEConfig, MoEModel  # noqa: E402
from paper_2310_18859_b200.offload import ExpertStore  # noqa: E402
from paper_2310_18859_b200.predictor import DeviceTable  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--tokens", type=int, default=32768)
p.add_argument("--experts", type=int, default=8)
p.add_argument("--d", type=int, default=768)
p.add_argument("--h", type=int, default=3072)
p.add_argument("--iters", type=int, default=20)
p.add_argument("--no-cublas", action="store_true")
p.add_argument("--exact", action="store_true", help="exactly tokens/experts rows per expert")
p.add_argument("--alias-slots", type=int, default=0,
               help="map every expert onto this many slots (weights L2-resident: isolates "
                    "the HBM weight stream)")
a = p.parse_args()
cfg = MoEConfig(vocab_size=64, d_model=a.d, num_layers=1, num_experts=a.experts,
                expert_hidden=a.h, max_seq_len=16)
model = MoEModel.synthetic(cfg, 0)
store = ExpertStore.full(model)
N, K = a.tokens, a.experts
ids = (torch.arange(N, device="cuda", dtype=torch.int32) % K).view(1, N, 1) if a.exact else \
    torch.randint(0, K, (1, N, 1), device="cuda", dtype=torch.int32)
al = torch.rand((1, N, 1), device="cuda", dtype=torch.float64)
dt = DeviceTable(ids, al, al.float(), N, 1)
dt.permute(K, torch.cuda.current_stream())
x = torch.randn(N, a.d, device="cuda")
torch.cuda.synchronize()
dt.ready.synchronize()
hist = dt.hist.cpu().numpy()
out = store.run_layer(model, 0, x, dt)  # loads experts
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
from paper_2310_18859_b200.offload import Wave, run_waves  # noqa: E402
need = [int(e) for e in np.nonzero(hist[0])[0]]
wave = Wave(0, [], need, store.slot_row(0, need))
if a.alias_slots:
    wave.slot_row = (wave.slot_row % a.alias_slots).astype(np.int32)
for _ in range(3):
    run_waves(model, [wave], x, dt, store, torch.cuda.current_stream())
torch.cuda.synchronize()
e0.record()
for _ in range(a.iters):
    run_waves(model, [wave], x, dt, store, torch.cuda.current_stream())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
fl = 4.0 * N * a.d * a.h
print(f"ffn layer: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s  (N={N}, K={K}, d={a.d}, h={a.h})")
if os.environ.get("SIDA_GEMM_PROF"):
    from paper_2310_18859_b200 import _lib
    buf = np.zeros((2, 148, 12), dtype=np.uint64)
    _lib.check(_lib.load().sida_debug_gemm_prof(buf.ctypes.data))
    names = ["prod_wait_empty", "mma_wait_epi", "mma_wait_tma", "mma_total", "epi_wait_full",
             "epi_total", "tiles"]
    for gi in range(2):
        b = buf[gi].astype(np.float64)
        lead = b[b[:, 3] > 0]
        if len(lead):
            print(f"GEMM{gi + 1} per issuing CTA: mma_total min {lead[:, 3].min():.0f} mean "
                  f"{lead[:, 3].mean():.0f} max {lead[:, 3].max():.0f}; epi_total min "
                  f"{b[:, 5].min():.0f} max {b[:, 5].max():.0f}; tiles {lead[:, 6].min():.0f}.."
                  f"{lead[:, 6].max():.0f} ({len(lead)} issuers)")
        ent, wt, ex = b[:, 8], b[:, 9], b[:, 10]
        t0 = buf[0][:, 8].astype(np.float64).min()
        print(f"GEMM{gi + 1} timeline (us from GEMM1's first CTA entry): entry {(ent.min() - t0) / 1e3:.1f}"
              f"..{(ent.max() - t0) / 1e3:.1f}, past PDL wait {(wt.min() - t0) / 1e3:.1f}.."
              f"{(wt.max() - t0) / 1e3:.1f}, exit {(ex.min() - t0) / 1e3:.1f}..{(ex.max() - t0) / 1e3:.1f}")
        tot = b[:, 3].mean()
        print(f"GEMM{gi + 1}: " + ", ".join(f"{n}={b[:, i].mean():.0f}" for i, n in enumerate(names))
              + f"  | mma waits epi {b[:, 1].mean() / tot:.1%} tma {b[:, 2].mean() / tot:.1%}")
if os.environ.get("SIDA_XFFN_PROF"):
    from paper_2310_18859_b200 import _lib
    buf = np.zeros((148, 8), dtype=np.uint64)
    _lib.check(_lib.load().sida_debug_xffn_prof(buf.ctypes.data_as(__import__("ctypes").c_void_p)))
    b = buf.astype(np.float64)
    lead = b[0::2]
    tot = lead[:, 4].mean()
    names = ["prod_wait_empty", "prod_wait_flag", "mma_wait_full", "mma_wait_chunk", "mma_total",
             "epi_wait_tile", "epi_total", "prologue"]
    print("xffn (leader CTAs, mean): " + ", ".join(f"{n}={lead[:, i].mean():.0f}"
                                                  for i, n in enumerate(names)))
    print(f"  mma waits: full {lead[:, 2].mean() / tot:.1%}, chunk {lead[:, 3].mean() / tot:.1%};"
          f" producer waits empty {lead[:, 0].mean() / tot:.1%}, flags {lead[:, 1].mean() / tot:.1%};"
          f" epilogue wait {lead[:, 5].mean() / tot:.1%}; mma_total spread "
          f"{lead[:, 4].min():.0f}..{lead[:, 4].max():.0f}")
if a.no_cublas:
    sys.exit(0)
# cuBLAS reference on the same shapes (dense bmm, no gather/epilogue fusion)
E = K
xs = torch.randn(E, N // E, a.d, device="cuda", dtype=torch.bfloat16)
w1 = torch.randn(E, a.d, a.h, device="cuda", dtype=torch.bfloat16)
w2 = torch.randn(E, a.h, a.d, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    torch.bmm(torch.bmm(xs, w1), w2)
torch.cuda.synchronize()
e0.record()
for _ in range(a.iters):
    hh = torch.bmm(xs, w1)
    torch.bmm(hh, w2)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(f"cuBLAS bmm pair: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s")
