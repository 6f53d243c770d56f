"""Rpotrf timing sweep (block width x mode x n) on one GPU: CUDA events
around the call on torch's current stream; prints dd GFlops (n^3/3, the
reference bench's count, mpkit/bench.py:68-69)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2109_13406_b200 import DeviceMatrix, Rpotrf  # noqa: E402


def spd_device(n, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    hi = torch.rand((n, n), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    lo = hi * (torch.rand((n, n), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * 2.0 ** -54
    hi = torch.tril(hi) + torch.tril(hi, -1).T
    lo = torch.tril(lo) + torch.tril(lo, -1).T
    hi.diagonal().add_(n + 1.0)
    lo.diagonal().zero_()
    return hi.T.contiguous().reshape(-1), lo.T.contiguous().reshape(-1)


def main():
    ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2048,4096,8192").split(",")]
    nbs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "64,128,256").split(",")]
    modes = (sys.argv[3] if len(sys.argv) > 3 else "fast,exact").split(",")
    for n in ns:
        h0, l0 = spd_device(n)
        for mode in modes:
            for nb in nbs:
                ts = []
                for rep in range(3):
                    a = DeviceMatrix(n, n, "dd", n, store=(h0.clone(), l0.clone()))
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    info = Rpotrf("L", n, a, n, mode=mode, nb=nb)
                    e1.record()
                    torch.cuda.synchronize()
                    assert info == 0, info
                    ts.append(e0.elapsed_time(e1) / 1e3)
                t = min(ts)
                print(f"n={n} mode={mode} nb={nb} t={t*1e3:.1f} ms  {n**3/3/t/1e9:.0f} GFlops", flush=True)


if __name__ == "__main__":
    main()
