"""Dev tool: does the fast kernel's speed depend on operand values?
Times Rgemm NN 8192^3 (fast) on random, constant and lo = 0 operands."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402

from paper_2109_13406_b200 import DeviceMatrix, Rgemm  # noqa: E402
from paper_2109_13406_b200.synth import hashed_dd_device  # noqa: E402

n = 8192
mode = sys.argv[1] if len(sys.argv) > 1 else "fast"


def mk(kind, tag):
    if kind == "random":
        h, l = hashed_dd_device(n, n, 7, tag, "cuda")
    elif kind == "const":
        h = torch.full((n * n,), 0.75, dtype=torch.float64, device="cuda")
        l = torch.full((n * n,), 0.75 * 2 ** -60, dtype=torch.float64, device="cuda")
    elif kind == "lo0":
        h, _ = hashed_dd_device(n, n, 7, tag, "cuda")
        l = torch.zeros_like(h)
    elif kind == "pow2":   # hi = +-2^e, lo = 0: products exact
        h, _ = hashed_dd_device(n, n, 7, tag, "cuda")
        h = torch.sign(h) * torch.exp2(torch.round(torch.log2(h.abs())))
        l = torch.zeros_like(h)
    return DeviceMatrix(n, n, "dd", n, store=(h, l))


for kind in ("random", "const", "lo0", "pow2"):
    A, B, C = mk(kind, 1), mk(kind, 2), mk(kind, 3)
    Rgemm("N", "N", n, n, n, 1.5, A, n, B, n, 0.5, C, n, mode=mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    Rgemm("N", "N", n, n, n, 1.5, A, n, B, n, 0.5, C, n, mode=mode)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(f"{mode} {kind:7s}: {t*1e3:8.2f} ms  {2*n**3/t/1e9:8.1f} dd GFlops", flush=True)
    del A, B, C
