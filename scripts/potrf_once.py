"""One warm Rpotrf call (for profilers): python potrf_once.py n nb mode [uplo]."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2109_13406_b200 import DeviceMatrix, Rpotrf  # noqa: E402
from scripts.potrf_time import spd_device  # noqa: E402

n, nb, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
uplo = sys.argv[4] if len(sys.argv) > 4 else "L"
h0, l0 = spd_device(n)
for rep in range(2):
    a = DeviceMatrix(n, n, "dd", n, store=(h0.clone(), l0.clone()))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    info = Rpotrf(uplo, n, a, n, mode=mode, nb=nb)
    t1 = time.perf_counter()
    print(f"rep {rep}: info={info} host {1e3 * (t1 - t0):.2f} ms", flush=True)
