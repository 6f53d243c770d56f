"""Dev tool: time one Rgemm shape.  python scripts/shape_time.py m n k [mode] [ta tb]"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402

from paper_2109_13406_b200 import DeviceMatrix, Rgemm  # noqa: E402
from paper_2109_13406_b200.synth import hashed_dd_device  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
mode = sys.argv[4] if len(sys.argv) > 4 else "fast"
ta, tb = (sys.argv[5], sys.argv[6]) if len(sys.argv) > 6 else ("N", "N")
nra, nca = (m, k) if ta == "N" else (k, m)
nrb, ncb = (k, n) if tb == "N" else (n, k)
A = DeviceMatrix(nra, nca, "dd", nra, store=hashed_dd_device(nra, nca, 1, 1, "cuda"))
B = DeviceMatrix(nrb, ncb, "dd", nrb, store=hashed_dd_device(nrb, ncb, 1, 2, "cuda"))
C = DeviceMatrix(m, n, "dd", m, store=hashed_dd_device(m, n, 1, 3, "cuda"))
Rgemm(ta, tb, m, n, k, 1.5, A, nra, B, nrb, 0.5, C, m, mode=mode)
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    Rgemm(ta, tb, m, n, k, 1.5, A, nra, B, nrb, 0.5, C, m, mode=mode)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
t = min(ts)
gf = 2.0 * m * n * k / t / 1e9
print(f"{mode} {ta}{tb} m={m} n={n} k={k}: {t*1e3:.2f} ms {gf:.1f} dd GFlops ({gf/3720*100:.1f}% roof)",
      flush=True)
