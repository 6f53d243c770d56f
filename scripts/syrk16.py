"""Time Rsyrk U/N (or Rgemm NN) at n = k on one GPU, two calls (the first pays
one-time pool growth): python scripts/syrk16.py n syrk|gemm"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2109_13406_b200 import DeviceMatrix, Rgemm, Rsyrk, flop_count  # noqa: E402
from paper_2109_13406_b200.synth import hashed_dd_device  # noqa: E402

n = int(sys.argv[1])
what = sys.argv[2]
A = DeviceMatrix(n, n, "dd", n, store=hashed_dd_device(n, n, 0, 1, "cuda"))
C = DeviceMatrix(n, n, "dd", n, store=hashed_dd_device(n, n, 0, 3, "cuda"))
B = DeviceMatrix(n, n, "dd", n, store=hashed_dd_device(n, n, 0, 2, "cuda")) if what == "gemm" else None
for it in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if what == "gemm":
        Rgemm("N", "N", n, n, n, 1.5, A, n, B, n, 0.5, C, n)
        f = 2.0 * n ** 3
    else:
        Rsyrk("U", "N", n, n, 1.5, A, n, 0.5, C, n)
        f = flop_count("Rsyrk", n, k=n)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(what, n, f"{t * 1e3:.1f} ms {f / t / 1e9:.1f} dd GFlops")
