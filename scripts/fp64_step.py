"""FP64-pipe lane operations of one bench step, from an ncu launch list.

    ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,\\
sm__inst_executed_pipe_tensor_subpipe_dmma.sum --clock-control none --csv \\
        --log-file gpurun_out/fp64_step.csv python bench.py --steps 1 --warmup 0 --quick
    python scripts/fp64_step.py gpurun_out/fp64_step.csv 8192 fast > profiles/r2_fp64_step.json

Counts every launch of the library's kernels in the capture except the live
DFMA peak probe (dfma_burn): with --steps 1 --warmup 0 that is exactly one
step.  Lane operations = 32 x FP64-pipe warp instructions (DFMA / DADD /
DMUL ...) + 256 x DMMA.8x8x4 instructions (each 8 x 8 x 4 multiply-adds on the
same FP64 pipe)."""
import collections
import csv
import json
import sys

path, n, mode = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
per = collections.defaultdict(lambda: collections.defaultdict(float))
for d in data:
    name = d["Kernel Name"]
    if "dfma_burn" in name:
        continue
    if not any(s in name for s in ("ddb", "tma::", "cross::", "tiled::", "umma::")):
        continue
    key = (d["ID"], name.split("(")[0][:80])
    v = float(d["Metric Value"].replace(",", "")) if d["Metric Value"] not in ("", "n/a") else 0.0
    per[key][d["Metric Name"]] = v
kern = collections.defaultdict(lambda: {"launches": 0, "fp64_inst": 0.0, "dmma_inst": 0.0,
                                        "ms": 0.0})
for (lid, name), m in per.items():
    k = kern[name]
    k["launches"] += 1
    k["fp64_inst"] += m.get("sm__inst_executed_pipe_fp64.sum", 0.0)
    k["dmma_inst"] += m.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0)
    k["ms"] += m.get("gpu__time_duration.sum", 0.0) / 1e6
lane = sum(32 * k["fp64_inst"] + 256 * k["dmma_inst"] for k in kern.values())
out = {"n": n, "mode": mode, "fp64_lane_ops_per_step": lane,
       "fp64_lane_ops_per_mac": lane / float(n) ** 3,
       "ncu_serialised_ms": sum(k["ms"] for k in kern.values()),
       "per_kernel": dict(sorted(kern.items(), key=lambda kv: -kv[1]["ms"])),
       "source": path,
       "how": "32 x sm__inst_executed_pipe_fp64.sum + 256 x "
              "sm__inst_executed_pipe_tensor_subpipe_dmma.sum over every library launch of "
              "one step (bench.py --steps 1 --warmup 0 --quick), dfma_burn excluded"}
print(json.dumps(out, indent=1))
