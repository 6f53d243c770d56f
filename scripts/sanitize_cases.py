"""Small ragged cases for compute-sanitizer (one tool per run):
    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
Covers every kernel family: exact / fast / twosum tiled (cp.async), the TMA NN
kernel, split-K, Rsyrk U/L, binary64, Cgemm cdd / c64, reference kernel."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_13406_b200 import Cgemm, DeviceMatrix, Rgemm, Rsyrk  # noqa: E402
from paper_2109_13406_b200.synth import random_dd  # noqa: E402


def dmat(rows, cols, ld, seed, tag, prec="dd"):
    hi, lo = random_dd(rows, cols, ld, seed, tag)
    t = lambda x: torch.from_numpy(x.copy()).cuda()
    if prec == "dd":
        return DeviceMatrix(rows, cols, "dd", ld, store=(t(hi), t(lo)))
    if prec == "f64":
        return DeviceMatrix(rows, cols, "f64", ld, store=(t(hi),))
    if prec == "cdd":
        h2, l2 = random_dd(rows, cols, ld, seed, tag + 10)
        return DeviceMatrix(rows, cols, "cdd", ld, store=(t(hi), t(lo), t(h2), t(l2)))
    return DeviceMatrix(rows, cols, "c64", ld, store=(torch.from_numpy((hi + 1j * lo * 1e15).copy()).cuda(),))


for prec, modes in (("dd", ("exact", "fast", "twosum", "reference")), ("f64", ("exact",))):
    for ta, tb in (("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")):
        for (m, n, k, pad) in ((37, 29, 41, 3), (130, 66, 1100, 0), (64, 64, 2048, 2)):
            nra, nca = (m, k) if ta == "N" else (k, m)
            nrb, ncb = (k, n) if tb == "N" else (n, k)
            a, b = dmat(nra, nca, nra + pad, 1, 1, prec), dmat(nrb, ncb, nrb + pad, 1, 2, prec)
            for mode in modes:
                c = dmat(m, n, m + pad, 1, 3, prec)
                Rgemm(ta, tb, m, n, k, 1.5, a, nra + pad, b, nrb + pad, 0.5, c, m + pad, mode=mode)
    for up in ("U", "L"):
        for tr in ("N", "T"):
            n, k = 131, 37
            nra, nca = (n, k) if tr == "N" else (k, n)
            a = dmat(nra, nca, nra + 1, 2, 1, prec)
            for mode in modes:
                c = dmat(n, n, n + 1, 2, 3, prec)
                Rsyrk(up, tr, n, k, 1.5, a, nra + 1, 0.5, c, n + 1, mode=mode)
for prec, modes in (("cdd", ("exact", "fast")), ("c64", ("exact",))):
    m, n, k = 33, 21, 19
    a, b = dmat(m, k, m + 1, 3, 1, prec), dmat(k, n, k, 3, 2, prec)
    for mode in modes:
        c = dmat(m, n, m, 3, 3, prec)
        Cgemm("C", "N", m, n, k, complex(1, 2), a if False else dmat(k, m, k, 3, 1, prec), k, b, k,
              0.5, c, m, mode=mode)
torch.cuda.synchronize()
print("sanitize cases done")
