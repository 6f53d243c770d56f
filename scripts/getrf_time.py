"""Rgetrf timing on one GPU: python scripts/getrf_time.py n1,n2 mode1,mode2
(random dd matrix; CUDA events; dd GFlops = 2n^3/3, mpkit/bench.py:66-67)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2109_13406_b200 import DeviceMatrix, Rgetrf  # noqa: E402
from paper_2109_13406_b200.synth import hashed_dd_device  # noqa: E402

ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2048,4096,8192").split(",")]
modes = (sys.argv[2] if len(sys.argv) > 2 else "fast,exact").split(",")
for n in ns:
    h0, l0 = hashed_dd_device(n, n, 0, 1, "cuda")
    for mode in modes:
        ts = []
        for rep in range(2):
            a = DeviceMatrix(n, n, "dd", n, store=(h0.clone(), l0.clone()))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ipiv, info = Rgetrf(n, n, a, n, mode=mode)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = min(ts)
        print(f"n={n} mode={mode} t={t*1e3:.1f} ms {2*n**3/3/t/1e9:.0f} GFlops info={info}", flush=True)
