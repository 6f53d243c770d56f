"""Dev tool: time every tiled accumulation algorithm on one shape and check
its accuracy on sampled entries against the exact-rational oracle.

    python scripts/variants.py [n] [k]
"""
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def run_child(alg, n, k, trans):
    env = dict(os.environ)
    parts = alg.split("@")          # alg[@tile[@libvariant]]
    alg = parts[0]
    tile = parts[1] if len(parts) > 1 and parts[1] else "big"
    if len(parts) > 2:
        env["DDBLAS_LIB"] = os.path.join(REPO, "scripts", "libs", f"libddblas_{parts[2]}.so")
        env["DDB_LIBTAG"] = parts[2]
    env["DDB_TILE"] = tile
    env["DDB_FAST_ALG"] = alg
    out = subprocess.run([sys.executable, __file__, "--child", alg, str(n), str(k), trans],
                         env=env, capture_output=True, text=True)
    sys.stdout.write(out.stdout)
    if out.returncode:
        sys.stdout.write(out.stderr[-3000:])


def child(alg, n, k, trans):
    from oracle import exact
    from paper_2109_13406_b200 import DeviceMatrix, Rgemm, _lib
    from paper_2109_13406_b200.synth import random_dd
    ta, tb = trans
    m = n
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A = random_dd(nra, nca, nra, 0, 1)
    B = random_dd(nrb, ncb, nrb, 0, 2)
    C = random_dd(m, n, m, 0, 3)
    dev = lambda r, c, P: DeviceMatrix(r, c, "dd", r, store=tuple(torch.from_numpy(p).cuda() for p in P))
    a, b = dev(nra, nca, A), dev(nrb, ncb, B)
    c0 = dev(m, n, C)
    c = c0.copy()
    mode = "exact" if alg == "exact" else "fast"   # DDB_FAST_ALG picks the fast kernel
    alpha, beta = 1.5, 0.5
    Rgemm(ta, tb, m, n, k, alpha, a, nra, b, nrb, beta, c, m, mode=mode)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        c = c0.copy()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        Rgemm(ta, tb, m, n, k, alpha, a, nra, b, nrb, beta, c, m, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t = min(times)
    gf = 2.0 * m * n * k / t / 1e9
    gh, gl = c.store[0].cpu().numpy(), c.store[1].cpu().numpy()
    I = list(range(0, m, m // 6))[:6]
    J = list(range(0, n, n // 6))[:6]
    vals, scales = exact.exact_entries(ta, tb, k, (1.5, 0.0), A[0], A[1], nra, B[0], B[1], nrb,
                                       (0.5, 0.0), C[0], C[1], m, I, J)
    try:
        worst = exact.error_ratios(gh, gl, m, I, J, vals, scales, k)
    except ValueError:
        worst = float("nan")
    print(f"{alg:8s} {os.environ.get('DDB_TILE','big'):5s} {os.environ.get('DDB_LIBTAG','main'):5s} {trans} n={n} k={k}: {t*1e3:9.2f} ms  {gf:9.1f} dd GFlops  "
          f"({gf/3720*100:5.1f}% of 3.72 TF roof)  err/bound {worst:.3e}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
    else:
        n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
        k = int(sys.argv[2]) if len(sys.argv) > 2 else n
        algs = sys.argv[3].split(",") if len(sys.argv) > 3 else ["cert", "twosum", "exact"]
        trans = sys.argv[4] if len(sys.argv) > 4 else "NN"
        for alg in algs:
            run_child(alg, n, k, trans)
