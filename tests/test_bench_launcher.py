"""CPU: bench.py's multi-GPU launcher.  `python bench.py --gpus N` outside
torchrun re-launches itself with N ranks (torch.distributed.run on
127.0.0.1); the --dry-run test hook runs the rank / timing / JSON plumbing
on gloo with a stand-in step, so the world-2 path is exercised without GPUs."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args,
                          capture_output=True, text=True, timeout=timeout, cwd=REPO, env=env)


def _json_lines(stdout):
    return [json.loads(x) for x in stdout.splitlines() if x.startswith("{")]


def test_self_launch_runs_two_ranks_and_reports_world_two():
    out = _run(["--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "1"])
    assert out.returncode == 0, out.stderr[-3000:]
    lines = _json_lines(out.stdout)
    assert len(lines) == 1, out.stdout           # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2 and lines[0]["dry_run"] is True
    assert lines[0]["steps"] == 2 and lines[0]["ms_per_step"] > 0


def test_single_rank_dry_run_reports_one():
    out = _run(["--gpus", "1", "--dry-run", "--steps", "1", "--warmup", "1"])
    assert out.returncode == 0, out.stderr[-3000:]
    assert _json_lines(out.stdout)[0]["n_gpus"] == 1


def test_refuses_more_gpus_than_visible():
    """Asking for more GPUs than the box has fails loudly instead of quietly
    measuring one GPU (this container has none)."""
    import torch
    if torch.cuda.device_count() >= 2:
        return
    out = _run(["--gpus", "2", "--steps", "1", "--warmup", "1"], timeout=300)
    assert out.returncode == 2
    line = _json_lines(out.stdout)[0]
    assert "error" in line and line["n_gpus"] < 2
