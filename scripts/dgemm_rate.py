"""cuBLAS DGEMM (binary64, torch.matmul) throughput on this GPU at n^3, to
size a split of the fast dd MAC into an anchored hi*hi kernel plus the
lo*hi + hi*lo cross terms as two plain DGEMMs.  Usage: dgemm_rate.py [n]"""
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = torch.empty(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = min(ts)
print(f"dgemm n={n}: {t:.2f} ms  {2 * n ** 3 / t / 1e9:.1f} TFLOP/s  all={['%.2f' % x for x in ts]}")
# accuracy spot check against a dd-exact-ish reference on a corner block
r = (a[:64].to(torch.float64) @ b[:, :64])
print("max |diff| corner:", float((r - c[:64, :64]).abs().max()))
