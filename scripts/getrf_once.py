"""One warm Rgetrf call (for profilers / DDB_LAPACK_TRACE): getrf_once.py n mode"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2109_13406_b200 import DeviceMatrix, Rgetrf  # noqa: E402
from paper_2109_13406_b200.synth import hashed_dd_device  # noqa: E402

n, mode = int(sys.argv[1]), sys.argv[2]
h0, l0 = hashed_dd_device(n, n, 0, 1, "cuda")
for rep in range(2):
    a = DeviceMatrix(n, n, "dd", n, store=(h0.clone(), l0.clone()))
    torch.cuda.synchronize()
    ipiv, info = Rgetrf(n, n, a, n, mode=mode)
    torch.cuda.synchronize()
    print(f"rep {rep}: info={info}", flush=True)
