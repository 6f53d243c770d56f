"""Benchmark: dd GFlops of Rgemm (2mnk) / Rsyrk (n(n+1)k) at n = 8192 on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--n 8192] [--mode fast|exact|twosum]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

Metric (BASELINE.json): "dd GFlops (Rgemm 2mnk, Rsyrk n(n+1)k) at n=8192,
1/2/4/8 B200 vs FP64 roof".  One step = one dd Rgemm NN, m = n = k = 8192,
alpha = 1.5, beta = 0.5, seeded random dd operands (hi ~ U(-1,1), lo ~ 2^-53
hi; paper_2109_13406_b200/synth.py) resident in HBM: 3 GiB of operands, far
larger than the 126 MB L2, so no flush is needed between steps.  At N > 1 the
same total problem is split by column blocks of C over the ranks (strong
scaling): A is broadcast from rank 0 over NCCL, B / C column blocks are
scattered and C gathered back, all inside the timed region
(paper_2109_13406_b200/parallel.py).

Printed keys beyond the driver contract:
  roofline      FP64-pipe roofline of the dominant kernel (20 fp64 flops per
                dd MAC, the north star's convention; peak = DFMA rate measured
                live on this GPU by ddb_fp64_peak_probe)
  cpu_baseline  the reference algorithm on this box's host cores (the C port
                in oracle/, bit-identical to the reference), sampled
  e2e           the same Rgemm through the public API with pinned HOST
                buffers (H2D of A, B, C and D2H of C inside the timed region)
  rsyrk         Rsyrk U/N at n = k = 8192 (the metric's second routine)
  modes         exact (bit-identical) and twosum (no bound GEMM) at the same shape
"""

from __future__ import annotations

import argparse
import math
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "dd GFlops (Rgemm 2mnk, Rsyrk n(n+1)k) at n=8192, 1/2/4/8 B200 vs FP64 roof"
UNIT = "dd GFlops"
ALPHA, BETA = 1.5, 0.5


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=8192)
    p.add_argument("--mode", default="fast", choices=["fast", "exact", "twosum"])
    p.add_argument("--quick", action="store_true", help="skip the secondary measurements")
    p.add_argument("--force-dist", action="store_true",
                   help="use the distributed (NCCL) path even with one rank (testing)")
    p.add_argument("--dry-run", action="store_true",
                   help="TEST HOOK: launcher / ranks / timing / JSON plumbing only, on the CPU "
                        "(gloo, a stand-in numpy step); never a measurement")
    return p.parse_args()


# --------------------------------------------------------------------------
# N > 1 without torchrun: re-launch this script with one rank per GPU

def self_launch(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec under
    torch.distributed.run with N local ranks on 127.0.0.1 and return its exit
    code.  Refuses (exit 2) when fewer than N GPUs are visible, so a request
    for N GPUs never reports n_gpus = 1."""
    if not args.dry_run:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {have} "
                              "CUDA device(s) visible", "n_gpus": have}), flush=True)
            return 2
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args):
    """TEST HOOK (--dry-run): the multi-rank plumbing of run_ours on the CPU --
    gloo process group, barrier + max-over-ranks timing, rank 0's JSON line --
    with a stand-in numpy step instead of the GPU kernels."""
    import numpy as np
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    if world > 1:
        dist.init_process_group("gloo")
    x = np.random.default_rng(rank).standard_normal((128, 128))
    step = lambda: x @ x  # noqa: E731  (stand-in work, not a measurement)
    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
                          "dry_run": True, "data": "stand-in CPU step (test hook)"}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------------------
# clocks during the timed region

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None,
                "samples": len(self.rows), "reasons": reasons}


# --------------------------------------------------------------------------
# reference arm and CPU baseline: the oracle port of the reference algorithm

def cpu_sample_rate(n, k, cols, threads):
    """Time the reference algorithm (bit-exact C port, oracle/dd_oracle.c) on
    an m = n x cols x k sub-problem of the Rgemm NN workload; returns
    (dd GFlops, seconds, description)."""
    from oracle import oracle
    from paper_2109_13406_b200.synth import random_dd
    m = n
    A = random_dd(m, k, m, 0, 1)
    B = random_dd(k, cols, k, 0, 2)
    C = random_dd(m, cols, m, 0, 3)
    ch, cl = C[0].copy(), C[1].copy()
    t0 = time.perf_counter()
    rc = oracle.rgemm("N", "N", m, cols, k, (ALPHA, 0.0), A[0], A[1], m, B[0], B[1], k,
                      (BETA, 0.0), ch, cl, m, threads=threads)
    dt = time.perf_counter() - t0
    assert rc == 0
    return 2.0 * m * cols * k / dt / 1e9, dt, f"Rgemm NN m={m} n={cols} k={k} (columns of the n={n} workload)"


def cpu_sample_cols(n, k, seconds):
    """Columns of the n x n x k workload that take about `seconds` on the
    host cores, from a 16-column probe: a bounded sample (the whole-workload
    CPU run would take hours), rounded to a multiple of the thread count."""
    from oracle import oracle
    threads = max(1, oracle.max_threads())
    _, dt, _ = cpu_sample_rate(n, k, 16, 0)
    cols = int(16 * seconds / max(dt, 1e-3))
    cols = max(threads, (cols // threads) * threads)
    return min(cols, n)


def cpu_lapack_rates(n=512):
    """The reference's LAPACK consumers on the host (the bit-exact C port of
    the unblocked algorithms, one core) at a sample size n: dd GFlops in the
    reference bench's counting, for the rpotrf / rgetrf / rtrsm lines."""
    from oracle import oracle
    from paper_2109_13406_b200 import flop_count
    from paper_2109_13406_b200.synth import random_dd, spd_dd
    out = {}
    h, l = spd_dd(n, n, seed=0)
    t0 = time.perf_counter()
    oracle.rpotrf("L", n, h, l, n)
    out["rpotrf"] = flop_count("Rpotrf", n) / (time.perf_counter() - t0) / 1e9
    h, l = random_dd(n, n, n, 0, 1)
    t0 = time.perf_counter()
    oracle.rgetrf(n, n, h, l, n)
    out["rgetrf"] = flop_count("Rgetrf", n) / (time.perf_counter() - t0) / 1e9
    ah, al = random_dd(n, n, n, 0, 4)
    ah[:: n + 1] += 4.0
    bh, bl = random_dd(n, n, n, 0, 5)
    t0 = time.perf_counter()
    oracle.rtrsm("L", "L", "N", "N", n, n, (1.5, 0.0), ah, al, n, bh, bl, n)
    out["rtrsm"] = 1.0 * n ** 3 / (time.perf_counter() - t0) / 1e9
    return {k: {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"n={n}, unblocked reference order (oracle/dd_oracle.c)"}
            for k, v in out.items()}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle
    threads = oracle.max_threads()
    n = args.n
    cols = cpu_sample_cols(n, n, 2.0)
    for _ in range(args.warmup):
        cpu_sample_rate(n, n, cols, threads)
    rates, secs = [], []
    for _ in range(args.steps):
        r, dt, desc = cpu_sample_rate(n, n, cols, threads)
        rates.append(r)
        secs.append(dt)
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(secs) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64x2 (double-double)",
        "data": "synthetic", "config": {"workload": f"dd Rgemm NN m=n=k={n}", "n": n,
                                        "sample": desc, "flush": "inputs > L2 (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm

def device_operands(n, k, dev):
    import torch
    from paper_2109_13406_b200 import DeviceMatrix
    from paper_2109_13406_b200.synth import random_dd
    mats = []
    for rows, cols, tag in ((n, k, 1), (k, n, 2), (n, n, 3)):
        hi, lo = random_dd(rows, cols, rows, 0, tag)
        mats.append(DeviceMatrix(rows, cols, "dd", rows, store=(
            torch.from_numpy(hi).to(dev), torch.from_numpy(lo).to(dev))))
    return mats


def timed(fn, steps, warmup, stream, reset=None):
    import torch
    for _ in range(warmup):
        if reset:
            reset()
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        if reset:
            reset()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    return times


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2109_13406_b200 import HostMatrix, Rgemm, Rsyrk, _lib, flop_count
    from paper_2109_13406_b200 import parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = world > 1 or args.force_dist
    if distributed:
        # one CTA per tile in the GEMMs (read at the library's first launch):
        # the k-panel broadcasts' NCCL kernels need SMs while a panel's GEMM
        # runs, which the persistent walk would hold until it ends
        os.environ.setdefault("DDB_TMA_PERSISTENT", "0")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    n = k = args.n
    mode = args.mode
    stream = torch.cuda.current_stream(dev)
    flops = flop_count("Rgemm", n, k=k, m=n)

    if rank == 0 or not distributed:
        A, B, C0 = device_operands(n, k, dev)
        C = C0.copy()
    else:
        A = B = C0 = C = None

    def reset():
        if C is not None:
            C.store[0].copy_(C0.store[0])
            C.store[1].copy_(C0.store[1])

    if distributed:
        plan = parallel.RgemmPlan(n, n, k, world, rank, dev)

        def step():
            parallel.rgemm_columns(plan, "N", "N", ALPHA, A, B, BETA, C, mode=mode)
    else:
        def step():
            Rgemm("N", "N", n, n, k, ALPHA, A, n, B, k, BETA, C, n, mode=mode)

    launches0 = _lib.launch_count()
    with ClockSampler(local) as clocks:
        if distributed:
            dist.barrier()
        times = timed(step, args.steps, args.warmup, stream, reset)
    launches = _lib.launch_count() - launches0
    t_local = statistics.median(times)
    t = t_local
    if distributed:
        tt = torch.tensor([t_local], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    value = flops / t / 1e9

    extra = {}
    if rank == 0:
        # ---- roofline: the FP64 pipe (DFMA + DMMA share it) ----
        peak = _lib.fp64_peak_probe()        # DFMA lane-ops/s * 2, measured live
        kernel_t = t if not distributed else t_local
        share = world if distributed else 1
        macs = float(n) * n * k / share
        prof = _profile_traffic()
        fp64 = _profile_fp64_step()
        split_on = mode == "fast" and os.environ.get("DDB_SPLIT", "1") != "0"
        traffic = prof.get("dram_bytes_per_launch")
        try:
            with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
                hbm_peak = float(json.load(f)["hbm_gbs"])
        except Exception:
            hbm_peak = None
        lane_peak = peak / 2.0                   # FP64 FMA lane-ops per second
        # the hardware fraction of the whole step: FP64-pipe lane operations
        # issued per step (ncu: 32 x sm__inst_executed_pipe_fp64 + 256 x
        # DMMA.8x8x4 instructions, summed over every launch of one step,
        # profiles/r2_fp64_step.json) / step time / the pipe's lane rate
        lane_ops = None
        if fp64 and fp64.get("n") == n and fp64.get("mode") == mode and not distributed:
            lane_ops = fp64["fp64_lane_ops_per_step"]
        hw_frac = lane_ops / kernel_t / lane_peak if lane_ops else None
        dd_conv = 20.0 * macs / kernel_t / 1e12          # the north star's convention
        extra["roofline"] = {
            "bound": "fp64", "unit": "TFLOP/s",
            "achieved": (2.0 * lane_ops / kernel_t / 1e12) if lane_ops else None,
            "peak": peak / 1e12,
            "frac": hw_frac,
            "frac_source": ("ncu FP64-pipe lane ops per step (profiles/r2_fp64_step.json) / "
                            "CUDA-event step time / live DFMA peak") if hw_frac else None,
            "traffic": traffic,
            "frac_dd_convention": dd_conv * 1e12 / peak,
            "achieved_dd_convention": dd_conv,
            "convention": "20 fp64 flops per dd MAC (north star); peak = live DFMA probe",
            "fp64_instr_per_mac_measured": (lane_ops / macs) if lane_ops else None,
            "fp64_instr_split": ({"tma_kernel_hi_hi": 4.75, "cross_dmma": 2.0}
                                 if split_on else None),
            "algorithmic_bytes": 16.0 * (2 * n * k + 2 * n * n),
            # achieved DRAM bandwidth of the dominant kernel (ncu bytes / step time)
            # against the measured copy bandwidth
            "hbm_gbs": (traffic / kernel_t / 1e9) if traffic and not distributed else None,
            "hbm_peak_gbs": hbm_peak,
        }
        if not distributed:
            # accuracy of the timed result (checker, outside the timed region)
            extra["accuracy"] = _accuracy(n, k, A, B, C0, C, mode)
    if rank == 0 and not args.quick:
        # ---- e2e through the public API with pinned host buffers ----
        extra["e2e"] = _e2e(n, k, mode, distributed, world, rank, dev)
        # ---- Rsyrk U/N at n = k ----
        if not distributed:
            extra["rsyrk"] = _rsyrk(n, k, mode, dev, stream, max(1, args.steps // 2))
            extra["modes"] = _modes(n, k, dev, stream, A, B, C, C0, mode)
            extra["f64"] = _f64(n, dev, stream)
            extra["cgemm"] = _cgemm(n // 2, dev, stream, mode)
            extra["trans_sweep"] = _trans_sweep(n // 2, dev, stream, mode)
            extra["syrk_sweep"] = _syrk_sweep(n // 2, dev, stream, mode)
            extra["deep_k"] = _deep_k(n // 4, 8 * n, dev, stream, mode)
            extra["rpotrf"] = _rpotrf(n, dev, stream, mode)
            extra["rgetrf"] = _rgetrf(n, dev, stream, mode)
            extra["rtrsm"] = _rtrsm(n, dev, stream, mode)
        extra["config5"] = _config5(mode, dev, stream, distributed, world, rank)
        if not distributed:
            cpu_lp = cpu_lapack_rates()
            for key in ("rpotrf", "rgetrf", "rtrsm"):
                if key in extra:
                    extra[key]["cpu_baseline"] = cpu_lp[key]
                    # dd roof = measured DFMA peak / 20 fp64 flops per dd MAC x 2 dd flops
                    roof = extra["roofline"]["peak"] * 1e3 / 10.0
                    extra[key]["roofline_frac"] = extra[key]["value"] / roof
        cpu_rate, cpu_s, desc = cpu_sample_rate(n, k, cpu_sample_cols(n, k, 10.0), 0)
        from oracle import oracle
        extra["cpu_baseline"] = {"value": cpu_rate, "unit": UNIT, "cores": oracle.max_threads(),
                                 "kind": "port", "sample": desc, "seconds": cpu_s}
    elif distributed and not args.quick:
        _e2e(n, k, mode, distributed, world, rank, dev)
        _config5(mode, dev, stream, distributed, world, rank)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64x2 (double-double)", "data": "synthetic",
            "config": {"workload": f"dd Rgemm NN m=n=k={n}", "m": n, "n": n, "k": k,
                       "alpha": ALPHA, "beta": BETA, "mode": mode,
                       "parallelism": f"columns{world}" if distributed else "single",
                       "flush": "operands 3 GiB > 126 MB L2"},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "step_ms_all": [x * 1e3 for x in times],
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


def _profile_fp64_step():
    """FP64-pipe lane operations of one step (every launch), from the ncu
    capture committed under profiles/ (scripts/fp64_step.py)."""
    try:
        with open(os.path.join(REPO, "profiles", "r2_fp64_step.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _accuracy(n, k, A, B, C0, C, mode, rows=8, cols=8):
    """Error of sampled entries of the timed result against exact rationals
    (oracle/exact.py: the CHECKER, run after the timed region; 8 x 8 entries,
    full k), with mpmath at 240 bits on two of them.  Returns the max of
    |err| / (4 k 2^-104 (|alpha| sum|ab| + |beta| |c|)) and of |err| / |C|."""
    import numpy as np
    from oracle import exact
    g = np.random.default_rng(12345)
    I = sorted(g.choice(n, rows, replace=False).tolist())
    J = sorted(g.choice(n, cols, replace=False).tolist())
    ah = np.stack([A.store[0][i::n][:k].cpu().numpy() for i in I])
    al = np.stack([A.store[1][i::n][:k].cpu().numpy() for i in I])
    bh = np.stack([B.store[0][j * k:(j + 1) * k].cpu().numpy() for j in J])
    bl = np.stack([B.store[1][j * k:(j + 1) * k].cpu().numpy() for j in J])
    ch0 = np.array([[float(C0.store[0][i + j * n]) for j in J] for i in I])
    cl0 = np.array([[float(C0.store[1][i + j * n]) for j in J] for i in I])
    gh = np.array([[float(C.store[0][i + j * n]) for j in J] for i in I])
    gl = np.array([[float(C.store[1][i + j * n]) for j in J] for i in I])
    # the sampled sub-problem, rows I of op(A) (ld = rows) and columns J of op(B)
    R, Q = len(I), len(J)
    vals, scales = exact.exact_entries(
        "N", "N", k, (ALPHA, 0.0), ah.T.reshape(-1), al.T.reshape(-1), R,
        bh.reshape(-1), bl.reshape(-1), k, (BETA, 0.0), ch0.T.reshape(-1), cl0.T.reshape(-1), R,
        list(range(R)), list(range(Q)))
    ratio = exact.error_ratios(gh.T.reshape(-1), gl.T.reshape(-1), R, list(range(R)),
                               list(range(Q)), vals, scales, k, c=4.0)
    from fractions import Fraction
    rel = 0.0
    for x in range(R):
        for y in range(Q):
            v = vals[x][y]
            err = abs(Fraction(gh[x, y]) + Fraction(gl[x, y]) - v)
            if v != 0:
                rel = max(rel, float(err / abs(v)))
    mp = [float(exact.mp_check(vals[x][x], gh[x, x], gl[x, x])) for x in range(2)]
    return {"entries": R * Q, "k": k, "mode": mode, "max_err_over_bound": ratio,
            "bound": "4 k 2^-104 (|alpha| sum|a b| + |beta| |c|)",
            "max_rel_err": rel, "rel_bound_k_2^-104": k * 2.0 ** -104,
            "mpmath240_abs_err_first2": mp,
            "checker": "oracle/exact.py (exact rationals; mpmath 240-bit cross-check)"}


def _profile_traffic():
    """dram bytes per launch of the tiled kernel from the committed ncu
    capture (profiles/), if present."""
    path = os.path.join(REPO, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


def _shm_room(nbytes):
    try:
        st = os.statvfs("/dev/shm")
        return st.f_bavail * st.f_frsize > nbytes * 1.1
    except OSError:
        return False


def _e2e(n, k, mode, distributed, world, rank, dev):
    """The same Rgemm through the public API from pinned HOST planes, host
    copies inside the timed region.  N = 1: ddb_rgemm_host (copies pipelined
    with the kernels).  N > 1: every rank runs that host entry on its column
    slab, reading A / its B columns and writing its C columns through its OWN
    PCIe link from host planes in shared memory (parallel.rgemm_host_shared);
    without room in /dev/shm, rank 0 stages everything and the slabs go over
    NCCL (parallel.rgemm_host_columns)."""
    import torch
    from paper_2109_13406_b200 import HostMatrix, Rgemm
    from paper_2109_13406_b200 import parallel
    from paper_2109_13406_b200.matrix import SharedHostMatrix
    from paper_2109_13406_b200.synth import random_dd
    dims = ((n, k, 1), (k, n, 2), (n, n, 3))
    shared = False
    hm = []
    if distributed:
        import torch.distributed as dist
        flag = [_shm_room(16 * (n * k + k * n + n * n))] if rank == 0 else [None]
        dist.broadcast_object_list(flag, src=0)
        shared = bool(flag[0])
    if shared:
        names = [None] * 3
        if rank == 0:
            for rows, cols, tag in dims:
                m_ = SharedHostMatrix(rows, cols, "dd", rows, create=True)
                hi, lo = random_dd(rows, cols, rows, 0, tag)
                m_.store[0][:] = hi
                m_.store[1][:] = lo
                hm.append(m_)
            names = [x.name for x in hm]
        dist.broadcast_object_list(names, src=0)
        if rank != 0:
            hm = [SharedHostMatrix(rows, cols, "dd", rows, name=nm)
                  for (rows, cols, _), nm in zip(dims, names)]
        for x in hm:
            x.pin()                      # page-lock this rank's mapping (setup)
    elif rank == 0:
        for rows, cols, tag in dims:
            m_ = HostMatrix(rows, cols, "dd", rows, pinned=True)
            hi, lo = random_dd(rows, cols, rows, 0, tag)
            m_.store[0][:] = hi
            m_.store[1][:] = lo
            hm.append(m_)
    steps = 2
    times = []
    for it in range(steps + 1):
        torch.cuda.synchronize()
        if distributed:
            import torch.distributed as dist
            dist.barrier()
        t0 = time.perf_counter()
        if shared:
            parallel.rgemm_host_shared("N", "N", n, n, k, ALPHA, hm[0], hm[1], BETA, hm[2],
                                       world, rank, mode=mode)
        elif distributed:
            a, b, c = hm if hm else (None,) * 3
            parallel.rgemm_host_columns("N", "N", n, n, k, ALPHA, a, b, BETA, c, world, rank, dev,
                                        mode=mode)
        else:
            Rgemm("N", "N", n, n, k, ALPHA, hm[0], n, hm[1], k, BETA, hm[2], n, mode=mode)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if it:
            times.append(dt)
    t = statistics.median(times)
    if distributed:
        import torch.distributed as dist
        tt = torch.tensor([t], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        dist.barrier()
    if shared:
        for x in hm:
            x.close()
    w = n // max(1, world)
    return {"value": 2.0 * n * n * k / t / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": 16 * (n * k + k * n + n * n) + (16 * n * k * (world - 1)
                                                                   if shared else 0),
            "d2h_bytes_per_step": 16 * n * n,
            "ms_per_step": t * 1e3,
            "host_buffers": ("shared-memory host planes, pinned per rank; every rank runs "
                             "ddb_rgemm_host on its column slab over its own PCIe link "
                             "(parallel.rgemm_host_shared)" if shared else
                             "pinned numpy planes, " + (
                                 "parallel.rgemm_host_columns (staged on the root, then "
                                 "column-split)" if distributed else "ddb_rgemm_host")),
            "per_rank_slab_columns": w if distributed else n}


def _config5(mode, dev, stream, distributed, world, rank, n=32768):
    """BASELINE configs[4]: Rgemm NN and Rsyrk U/N at n = k = 32768 (48 GiB /
    32 GiB of operands), one warm-up and one timed call each (~15 s / ~8 s on
    one B200); at N > 1 through the
    column-split NCCL path (A broadcast in k-panels, B / C slabs P2P)."""
    import torch
    from paper_2109_13406_b200 import DeviceMatrix, Rgemm, Rsyrk, flop_count
    from paper_2109_13406_b200 import parallel
    from paper_2109_13406_b200.synth import hashed_dd_device
    out = {"workload": f"dd Rgemm NN and Rsyrk U/N at n=k={n}", "unit": UNIT, "mode": mode,
           "n_gpus": world, "steps": 1, "warmup": 1}
    mats = None
    if rank == 0 or not distributed:
        mats = [DeviceMatrix(n, n, "dd", n, store=hashed_dd_device(n, n, 0, t, dev))
                for t in (1, 2, 3)]
    A, B, C = mats if mats else (None,) * 3

    def sync_time(fn):
        fn()   # one warm-up call: the first call at a new size grows the workspace pools
        if distributed:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        if distributed:
            import torch.distributed as dist
            tt = torch.tensor([t], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    if distributed:
        plan = parallel.RgemmPlan(n, n, n, world, rank, dev)
        t = sync_time(lambda: parallel.rgemm_columns(plan, "N", "N", ALPHA, A, B, BETA, C,
                                                     mode=mode))
        del plan
    else:
        t = sync_time(lambda: Rgemm("N", "N", n, n, n, ALPHA, A, n, B, n, BETA, C, n, mode=mode))
    out["rgemm"] = {"value": 2.0 * n ** 3 / t / 1e9, "ms": t * 1e3}
    if distributed:
        t = sync_time(lambda: parallel.rsyrk_columns(n, n, world, rank, dev, "U", "N", ALPHA, A,
                                                     BETA, C, mode=mode))
    else:
        t = sync_time(lambda: Rsyrk("U", "N", n, n, ALPHA, A, n, BETA, C, n, mode=mode))
    out["rsyrk"] = {"value": flop_count("Rsyrk", n, k=n) / t / 1e9, "ms": t * 1e3}
    del A, B, C, mats
    torch.cuda.empty_cache()
    return out


def _rsyrk(n, k, mode, dev, stream, steps):
    import torch
    from paper_2109_13406_b200 import DeviceMatrix, Rsyrk, flop_count
    from paper_2109_13406_b200.synth import random_dd
    hi, lo = random_dd(n, k, n, 0, 1)
    A = DeviceMatrix(n, k, "dd", n, store=(torch.from_numpy(hi).to(dev), torch.from_numpy(lo).to(dev)))
    hi, lo = random_dd(n, n, n, 0, 3)
    C = DeviceMatrix(n, n, "dd", n, store=(torch.from_numpy(hi).to(dev), torch.from_numpy(lo).to(dev)))
    times = timed(lambda: Rsyrk("U", "N", n, k, ALPHA, A, n, BETA, C, n, mode=mode), steps, 1, stream)
    t = statistics.median(times)
    return {"workload": f"dd Rsyrk U N n=k={n}", "value": flop_count("Rsyrk", n, k=k) / t / 1e9,
            "unit": UNIT, "ms_per_step": t * 1e3, "mode": mode}


def _f64(n, dev, stream):
    """binary64 Rgemm NN (the reference's 'f64' precision, bit-exact path)."""
    import torch
    from paper_2109_13406_b200 import DeviceMatrix, Rgemm
    from paper_2109_13406_b200.synth import hashed_dd_device
    mats = [DeviceMatrix(n, n, "f64", n, store=(hashed_dd_device(n, n, 0, t, dev)[0],))
            for t in (1, 2, 3)]
    times = timed(lambda: Rgemm("N", "N", n, n, n, ALPHA, mats[0], n, mats[1], n, BETA,
                                mats[2], n), 2, 1, stream)
    t = min(times)
    return {"workload": f"f64 Rgemm NN m=n=k={n}", "value": 2.0 * n ** 3 / t / 1e9,
            "unit": "GFlops (binary64)", "ms": t * 1e3}


def _trans_sweep(n, dev, stream, mode):
    """BASELINE configs[1]: Rgemm m = n = k over NN / NT / TN / TT."""
    from paper_2109_13406_b200 import DeviceMatrix, Rgemm
    from paper_2109_13406_b200.synth import hashed_dd_device
    mats = [DeviceMatrix(n, n, "dd", n, store=hashed_dd_device(n, n, 0, t, dev)) for t in (1, 2, 3)]
    out = {"workload": f"dd Rgemm m=n=k={n}", "unit": UNIT, "mode": mode}
    for ta in "NT":
        for tb in "NT":
            times = timed(lambda: Rgemm(ta, tb, n, n, n, ALPHA, mats[0], n, mats[1], n, BETA,
                                        mats[2], n, mode=mode), 2, 1, stream)
            out[ta + tb] = 2.0 * n ** 3 / min(times) / 1e9
    return out


def _syrk_sweep(n, dev, stream, mode):
    """BASELINE configs[2]: Rsyrk n = k over uplo U / L x trans N / T."""
    from paper_2109_13406_b200 import DeviceMatrix, Rsyrk, flop_count
    from paper_2109_13406_b200.synth import hashed_dd_device
    A = DeviceMatrix(n, n, "dd", n, store=hashed_dd_device(n, n, 0, 1, dev))
    C = DeviceMatrix(n, n, "dd", n, store=hashed_dd_device(n, n, 0, 3, dev))
    out = {"workload": f"dd Rsyrk n=k={n}", "unit": UNIT, "mode": mode}
    for uplo in "UL":
        for tr in "NT":
            times = timed(lambda: Rsyrk(uplo, tr, n, n, ALPHA, A, n, BETA, C, n, mode=mode),
                          2, 1, stream)
            out[uplo + tr] = flop_count("Rsyrk", n, k=n) / min(times) / 1e9
    return out


def _deep_k(m, k, dev, stream, mode):
    """BASELINE configs[3]: Rgemm NN m = n, deep k (accumulation depth)."""
    from paper_2109_13406_b200 import DeviceMatrix, Rgemm
    from paper_2109_13406_b200.synth import hashed_dd_device
    A = DeviceMatrix(m, k, "dd", m, store=hashed_dd_device(m, k, 0, 1, dev))
    B = DeviceMatrix(k, m, "dd", k, store=hashed_dd_device(k, m, 0, 2, dev))
    C = DeviceMatrix(m, m, "dd", m, store=hashed_dd_device(m, m, 0, 3, dev))
    times = timed(lambda: Rgemm("N", "N", m, m, k, ALPHA, A, m, B, k, BETA, C, m, mode=mode),
                  2, 1, stream)
    t = min(times)
    return {"workload": f"dd Rgemm NN m=n={m} k={k}", "value": 2.0 * m * m * k / t / 1e9,
            "unit": UNIT, "ms": t * 1e3, "mode": mode}


def _cgemm(n, dev, stream, mode):
    """complex double-double Cgemm NN ('cdd'), 8mnk real dd flops per call."""
    from paper_2109_13406_b200 import Cgemm, DeviceMatrix
    from paper_2109_13406_b200.synth import hashed_dd_device
    mats = []
    for t in (1, 2, 3):
        re = hashed_dd_device(n, n, 0, t, dev)
        im = hashed_dd_device(n, n, 0, t + 10, dev)
        mats.append(DeviceMatrix(n, n, "cdd", n, store=(re[0], re[1], im[0], im[1])))
    times = timed(lambda: Cgemm("N", "N", n, n, n, complex(1.5, -0.25), mats[0], n, mats[1], n,
                                complex(0.5, 0.125), mats[2], n, mode=mode), 2, 1, stream)
    t = min(times)
    return {"workload": f"cdd Cgemm NN m=n=k={n}", "value": 8.0 * n ** 3 / t / 1e9,
            "unit": "dd GFlops (8mnk)", "ms": t * 1e3, "mode": mode}


def _rpotrf(n, dev, stream, mode):
    """blocked dd Cholesky (lower) of an n x n SPD matrix; n^3/3 flops
    (the reference bench's count, mpkit/bench.py:68-69)."""
    import torch
    from paper_2109_13406_b200 import DeviceMatrix, Rpotrf, flop_count
    g = torch.Generator(device=dev).manual_seed(0)
    hi = torch.rand((n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1
    lo = hi * (torch.rand((n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1) * 2.0 ** -54
    hi = torch.tril(hi) + torch.tril(hi, -1).T
    lo = torch.tril(lo) + torch.tril(lo, -1).T
    hi.diagonal().add_(n + 1.0)
    lo.diagonal().zero_()
    h0, l0 = hi.T.contiguous().reshape(-1), lo.T.contiguous().reshape(-1)
    del hi, lo
    A = DeviceMatrix(n, n, "dd", n, store=(h0.clone(), l0.clone()))
    infos = []

    def reset():
        A.store[0].copy_(h0)
        A.store[1].copy_(l0)

    times = timed(lambda: infos.append(Rpotrf("L", n, A, n, mode=mode)), 2, 1, stream, reset=reset)
    t = min(times)
    return {"workload": f"dd Rpotrf L n={n} (SPD, diagonally dominant)",
            "value": flop_count("Rpotrf", n) / t / 1e9, "unit": UNIT, "ms": t * 1e3,
            "mode": mode, "info": max(infos)}


def _rgetrf(n, dev, stream, mode):
    """blocked dd LU with partial pivoting of a random n x n matrix; 2n^3/3
    flops (mpkit/bench.py:66-67)."""
    from paper_2109_13406_b200 import DeviceMatrix, Rgetrf, flop_count
    from paper_2109_13406_b200.synth import hashed_dd_device
    h0, l0 = hashed_dd_device(n, n, 0, 1, dev)
    A = DeviceMatrix(n, n, "dd", n, store=(h0.clone(), l0.clone()))
    infos = []

    def reset():
        A.store[0].copy_(h0)
        A.store[1].copy_(l0)

    times = timed(lambda: infos.append(Rgetrf(n, n, A, n, mode=mode)[1]), 2, 1, stream, reset=reset)
    t = min(times)
    return {"workload": f"dd Rgetrf n={n} (random, partial pivoting)",
            "value": flop_count("Rgetrf", n) / t / 1e9, "unit": UNIT, "ms": t * 1e3,
            "mode": mode, "info": max(infos)}


def _rtrsm(n, dev, stream, mode):
    """dd Rtrsm L,L,N,N with an n x n lower-triangular A and n right-hand
    sides; n^3 flops (n^2 n / 2 multiply-adds)."""
    import torch
    from paper_2109_13406_b200 import DeviceMatrix, Rtrsm
    from paper_2109_13406_b200.synth import hashed_dd_device
    ah, al = hashed_dd_device(n, n, 0, 4, dev)
    f = 2.0 ** -math.ceil(math.log2(n))      # off-diagonal row sums < 1 < diagonal
    ah.mul_(f)
    al.mul_(f)
    ah.view(n, n).diagonal().add_(4.0)      # column-major: the diagonal either way
    A = DeviceMatrix(n, n, "dd", n, store=(ah, al))
    b0 = hashed_dd_device(n, n, 0, 5, dev)
    B = DeviceMatrix(n, n, "dd", n, store=(b0[0].clone(), b0[1].clone()))

    def reset():
        B.store[0].copy_(b0[0])
        B.store[1].copy_(b0[1])

    times = timed(lambda: Rtrsm("L", "L", "N", "N", n, n, 1.5, A, n, B, n, mode=mode), 2, 1,
                  stream, reset=reset)
    t = min(times)
    del torch
    return {"workload": f"dd Rtrsm L,L,N,N m=n={n}", "value": 1.0 * n ** 3 / t / 1e9,
            "unit": UNIT, "ms": t * 1e3, "mode": mode}


def _modes(n, k, dev, stream, A, B, C, C0, mode):
    from paper_2109_13406_b200 import Rgemm
    out = {}
    for other in ("exact", "twosum", "fast"):
        if other == mode:
            continue
        times = timed(lambda: Rgemm("N", "N", n, n, k, ALPHA, A, n, B, k, BETA, C, n, mode=other),
                      1, 1, stream)
        t = min(times)
        out[other] = {"ms": t * 1e3, "value": 2.0 * n * n * k / t / 1e9, "unit": UNIT}
    if mode == "fast" and os.environ.get("DDB_SPLIT", "1") != "0":
        # fast mode without the split: the certified-anchor MAC entirely in the
        # hand-written kernel (7.5 FP64 instructions per MAC, no library GEMM)
        saved = os.environ.get("DDB_SPLIT")
        os.environ["DDB_SPLIT"] = "0"
        try:
            times = timed(lambda: Rgemm("N", "N", n, n, k, ALPHA, A, n, B, k, BETA, C, n,
                                        mode="fast"), 1, 1, stream)
        finally:
            if saved is None:
                os.environ.pop("DDB_SPLIT", None)
            else:
                os.environ["DDB_SPLIT"] = saved
        t = min(times)
        out["fast_nosplit"] = {"ms": t * 1e3, "value": 2.0 * n * n * k / t / 1e9, "unit": UNIT,
                               "what": "DDB_SPLIT=0: cross terms inside the dd kernel"}
    C.store[0].copy_(C0.store[0])
    C.store[1].copy_(C0.store[1])
    return out


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.dry_run:
        run_dry(args)
        return
    if args.impl == "reference":
        run_reference_arm(args)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
