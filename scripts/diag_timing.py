"""Per-step breakdown of one potrf diagonal-block kernel (diagnostics build:
scripts/build_variant.sh diagt -DDDB_DIAG_TIMING; run with
DDBLAS_LIB=scripts/libs/libddblas_diagt.so)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2109_13406_b200 import DeviceMatrix, Rpotrf  # noqa: E402
from scripts.potrf_time import spd_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
h0, l0 = spd_device(n)
for _ in range(2):
    a = DeviceMatrix(n, n, "dd", n, store=(h0.clone(), l0.clone()))
    assert Rpotrf("L", n, a, n, mode=os.environ.get("DIAG_MODE", "fast"), nb=64) == 0
torch.cuda.synchronize()
lib = ctypes.CDLL(os.environ["DDBLAS_LIB"])
buf = np.zeros((64, 8), dtype=np.int64)
assert lib.ddb_debug_diag_timing(buf.ctypes.data_as(ctypes.c_void_p)) == 0
t = buf - buf[0, 0]
col = t[:, 1] - t[:, 0]
piv = t[:, 2] - t[:, 1]
upd = t[:, 3] - t[:, 1]
step = np.diff(t[:, 0])
print("cycles per step: column phase + barrier %.0f, pivot %.0f, update (warp 1) %.0f, step %.0f"
      % (col[:-1].mean(), piv[:-1].mean(), upd[:-2].mean(), step.mean()))
print("total %d cycles" % (t[-1, 4]))
# pivot j+1 runs between stamps 1 and 2 of step j; its own stamps 5-7 are in row j+1
ss = buf[1:63, 5] - buf[:62, 1]; sq = buf[1:63, 6] - buf[1:63, 5]; dv = buf[1:63, 7] - buf[1:63, 6]
print("pivot parts: ssub+check %.0f, sqrt %.0f, reciprocal %.0f cycles" % (ss.mean(), sq.mean(), dv.mean()))
for j in (0, 1, 16, 32, 48, 62):
    print(j, t[j])
