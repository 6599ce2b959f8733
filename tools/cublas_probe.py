"""cuBLAS reference rates for the FFN shapes (batched per expert and dense), CUDA events."""
import torch
import sys
E = int(sys.argv[1]) if len(sys.argv) > 1 else 128
N, d, h = 32768, 768, 3072
xs = torch.randn(E, N // E, d, device="cuda", dtype=torch.bfloat16)
w1 = torch.randn(E, d, h, device="cuda", dtype=torch.bfloat16)
w2 = torch.randn(E, h, d, device="cuda", dtype=torch.bfloat16)
hh = torch.bmm(xs, w1)
def t(f, it=20):
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
fl = 2.0 * N * d * h
print(f"E={E} bmm1 {t(lambda: torch.bmm(xs, w1)):.4f} ms  bmm2 {t(lambda: torch.bmm(hh, w2)):.4f} ms  (each {fl/1e9:.0f} GFLOP)")
x = xs.reshape(N, d); W1 = w1[0]; H = hh.reshape(N, h); W2 = w2[0]
print(f"dense mm1 {t(lambda: x @ W1):.4f} ms  mm2 {t(lambda: H @ W2):.4f} ms")
