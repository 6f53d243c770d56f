"""Per-step breakdown of one Rgetrf panel kernel launch (CTA 0), diagnostics
build (scripts/build_variant.sh diagt -DDDB_DIAG_TIMING; run with
DDBLAS_LIB=scripts/libs/libddblas_diagt.so).  panel_timing.py n"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2109_13406_b200 import DeviceMatrix, Rgetrf  # noqa: E402
from paper_2109_13406_b200.synth import hashed_dd_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
h0, l0 = hashed_dd_device(n, n, 0, 1, "cuda")
os.environ["DDB_GETRF_NB"] = "64"
for _ in range(2):
    a = DeviceMatrix(n, 64, "dd", n, store=(h0[: n * 64].clone(), l0[: n * 64].clone()))
    Rgetrf(n, 64, a, n, mode="fast")
torch.cuda.synchronize()
lib = ctypes.CDLL(os.environ["DDBLAS_LIB"])
buf = np.zeros((64, 8), dtype=np.int64)
assert lib.ddb_debug_panel_timing(buf.ctypes.data_as(ctypes.c_void_p)) == 0
K = int(os.environ.get("PANEL_K", "7")); t = buf[:63, :K].astype(float)
d = np.diff(t, axis=1)
names = [n for n in os.environ.get("PANEL_NAMES", "wait,keys,row+rec,scale+upd,publish,arrive").split(",")]
print("mean cycles per step:", ", ".join(f"{nm} {v:.0f}" for nm, v in zip(names, d.mean(axis=0))))
print("step (k0 -> next k0): %.0f cycles" % np.diff(buf[:63, 0]).mean())
if os.environ.get("PANEL_K7"):
    print("warp 0 keys + row fetch (k1 -> k7): %.0f, waiting for the bulk (k7 -> k2): %.0f" % (
        (buf[1:63, 7] - buf[1:63, 1]).mean(), (buf[1:63, 2] - buf[1:63, 7]).mean()))
