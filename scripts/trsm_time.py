"""Rtrsm timing: python scripts/trsm_time.py n mode[,mode] [side uplo transa diag]
(n x n triangular A with damped off-diagonal, n right-hand sides; n^3 flops)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

n = int(sys.argv[1])
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fast"]
for mode in modes:
    r = bench._rtrsm(n, "cuda", torch.cuda.current_stream(), mode)
    print(mode, r, flush=True)
