"""NCCL-path self test (one process per GPU; also runs with a single rank).

    torchrun --nproc-per-node N scripts/dist_selftest.py     (or plain python: 1 rank)

Runs parallel.rgemm_columns / rsyrk_columns in exact mode and checks the root's
result bit for bit against the single-GPU Rgemm / Rsyrk on the same inputs.
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2109_13406_b200 import DeviceMatrix, Rgemm, Rsyrk, parallel  # noqa: E402
from paper_2109_13406_b200.synth import random_dd  # noqa: E402


def mat(rows, cols, seed, tag, dev):
    hi, lo = random_dd(rows, cols, rows, seed, tag)
    return DeviceMatrix(rows, cols, "dd", rows, store=(torch.from_numpy(hi).to(dev),
                                                       torch.from_numpy(lo).to(dev)))


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    ok = True
    for ta, tb, m, n, k in (("N", "N", 300, 517, 65), ("T", "T", 130, 129, 300), ("N", "T", 64, 700, 33)):
        nra, nca = (m, k) if ta == "N" else (k, m)
        nrb, ncb = (k, n) if tb == "N" else (n, k)
        if rank == 0:
            A, B, C = mat(nra, nca, 1, 1, dev), mat(nrb, ncb, 1, 2, dev), mat(m, n, 1, 3, dev)
            ref = C.copy()
            Rgemm(ta, tb, m, n, k, 1.5, A, nra, B, nrb, 0.5, ref, m, mode="exact")
        else:
            A = B = C = ref = None
        plan = parallel.RgemmPlan(m, n, k, world, rank, dev)
        parallel.rgemm_columns(plan, ta, tb, 1.5, A, B, 0.5, C, mode="exact")
        if rank == 0:
            same = all(torch.equal(C.store[i], ref.store[i]) for i in range(2))
            print(f"rgemm_columns {ta}{tb} {m}x{n}x{k} world={world}: {'OK' if same else 'MISMATCH'}")
            ok &= same
    for up, tr in (("U", "N"), ("L", "T")):
        n, k = 400, 50
        nra, nca = (n, k) if tr == "N" else (k, n)
        if rank == 0:
            A, C = mat(nra, nca, 2, 1, dev), mat(n, n, 2, 3, dev)
            ref = C.copy()
            Rsyrk(up, tr, n, k, 1.5, A, nra, 0.5, ref, n, mode="exact")
        else:
            A = C = ref = None
        parallel.rsyrk_columns(n, k, world, rank, dev, up, tr, 1.5, A, 0.5, C, mode="exact")
        if rank == 0:
            same = all(torch.equal(C.store[i], ref.store[i]) for i in range(2))
            print(f"rsyrk_columns {up}{tr} n={n} k={k} world={world}: {'OK' if same else 'MISMATCH'}")
            ok &= same
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
