"""Time the fast mode's building blocks alone through the C ABI's diagnostic
entry points (CUDA events, best of N after a warm-up):
    python scripts/kernel_time.py cross 8192 [reps]   -- ddb_cross_terms (DMMA)
    python scripts/kernel_time.py bound 8192 [reps]   -- ddb_abs_bound (tcgen05; includes copies)
"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2109_13406_b200 import _lib  # noqa: E402

what, n = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
L = _lib.load()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
g = torch.Generator(device="cuda").manual_seed(1)
ah = torch.rand(n * n, device="cuda", dtype=torch.float64, generator=g)
al = ah * 2.0 ** -60
bh = torch.rand(n * n, device="cuda", dtype=torch.float64, generator=g)
bl = bh * 2.0 ** -60
x = torch.empty(n * n, device="cuda", dtype=torch.float64)
st = torch.cuda.current_stream().cuda_stream
if what == "cross":
    call = lambda: L.ddb_cross_terms(n, n, n, P(ah), P(al), n, P(bh), P(bl), n, P(x), 0,  # noqa: E731
                                     ctypes.c_void_p(st))
    flops = 2 * 2 * n ** 3
else:
    re = torch.empty(n, device="cuda", dtype=torch.int32)
    ce = torch.empty(n, device="cuda", dtype=torch.int32)
    s = torch.empty(n * n, device="cuda", dtype=torch.float32)
    call = lambda: L.ddb_abs_bound(b"N", b"N", n, n, n, P(ah), n, P(bh), n, P(re), P(ce),  # noqa: E731
                                   P(s), None, None, ctypes.c_void_p(st))
    flops = 2 * n ** 3
rc = call()
assert rc == 0, _lib.last_error()
torch.cuda.synchronize()
best = 1e30
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call()
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"{what} n={n}: {best:.3f} ms  {flops / best / 1e9:.1f} TFLOP/s")
