"""Time the PYTHON reference itself on BASELINE configs[0] (dd Rgemm NN
m = n = k = 256, alpha 1.5, beta 0.5) in the build container, the way the
reference's own bench does it (mpkit/bench.py:276-287: one warm-up call, then
best of `reps` with the scratch C copied outside the timed region), at t = 1
(sequential Rgemm) and t = cores (Rgemm_par).  TEST / MEASUREMENT
INFRASTRUCTURE ONLY: /root/reference does not exist on the GPU box, so this
runs here and its output is committed as profiles/r2_python_reference_cpu.json.

    python oracle/time_python_reference.py > profiles/r2_python_reference_cpu.json
"""

from __future__ import annotations

import json
import os
import platform
import subprocess
import sys
import time

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def main(n=256, reps=3):
    sys.path.insert(0, REF)
    from mpkit.mpblas import Matrix, Rgemm
    from mpkit.mpblas.parallel import Rgemm_par
    from paper_2109_13406_b200.synth import random_dd
    from oracle import oracle
    A, B, C = (random_dd(n, n, n, 0, t) for t in (1, 2, 3))

    def mat(planes):
        m = Matrix(n, n, "dd")
        m.store[0][:] = planes[0]
        m.store[1][:] = planes[1]
        return m

    a, b = mat(A), mat(B)
    out = {"workload": f"dd Rgemm NN m=n=k={n}, alpha 1.5, beta 0.5 (BASELINE configs[0])",
           "unit": "dd GFlops (2mnk)", "method": "1 warm-up + best of %d, perf_counter, "
           "scratch C copied outside the timed region (mpkit/bench.py:276-287)" % reps,
           "host": platform.processor() or platform.machine(), "cores": os.cpu_count()}
    try:
        out["cpu_model"] = [l.split(":", 1)[1].strip() for l in
                            subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()
                            if l.startswith("Model name")][0]
    except Exception:
        pass
    flops = 2.0 * n ** 3
    for label, threads in (("t1", 1), ("t_cores", os.cpu_count())):
        def call(c):
            if threads == 1:
                Rgemm("N", "N", n, n, n, 1.5, a, n, b, n, 0.5, c, n)
            else:
                Rgemm_par("N", "N", n, n, n, 1.5, a, n, b, n, 0.5, c, n, t=threads)
        call(mat(C))
        best = None
        for _ in range(reps):
            c = mat(C)
            t0 = time.perf_counter()
            call(c)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        out[label] = {"threads": threads, "seconds": best, "value": flops / best / 1e9}
    # the bit-exact C port on the same cores, for comparison with bench.py's
    # reference arm (which runs the port on the GPU box's host)
    ch, cl = C[0].copy(), C[1].copy()
    t0 = time.perf_counter()
    oracle.rgemm("N", "N", n, n, n, (1.5, 0.0), A[0], A[1], n, B[0], B[1], n, (0.5, 0.0), ch, cl,
                 n, threads=0)
    dt = time.perf_counter() - t0
    out["c_port_all_cores"] = {"threads": oracle.max_threads(), "seconds": dt,
                               "value": flops / dt / 1e9}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
