"""Summarise an ncu report (raw page) into the numbers the roofline cites.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [label] > profiles/<name>.md
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv > profiles/<name>_launches.md
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active (% of peak)"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst executed (% of peak)"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
     "DMMA (FP64 tensor subpipe) inst executed (% of peak)"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active (% of elapsed)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (% of 64)"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid size"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(r, hdr, units) for r in rows[2:]]


def summarise(rep, label):
    lines = [f"# ncu summary: {label}", "", f"report: `{rep}` (ncu --set full --clock-control none)", ""]
    traffic = None
    for vals, hdr, units in raw(rep):
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        lines.append(f"## {d.get('Kernel Name', '?')[:120]}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for key, name in KEYS:
            if key in d:
                lines.append(f"| {name} (`{key}`) | {d[key]} | {u.get(key, '')} |")
        stalls = sorted(((float(d[h]), h[len(STALLS):].replace("_per_issue_active.ratio", ""))
                         for h in hdr if h.startswith(STALLS) and h.endswith("per_issue_active.ratio")
                         and d[h] not in ("", "n/a")), reverse=True)
        lines.append("")
        lines.append("stall reasons (warps per issue-active cycle): " +
                     ", ".join(f"{n} {v:.3f}" for v, n in stalls[:8]))
        lines.append("")
        try:
            rd = float(d["dram__bytes_read.sum"]) * (1e9 if u["dram__bytes_read.sum"] == "Gbyte" else 1e6 if u["dram__bytes_read.sum"] == "Mbyte" else 1)
            wr = float(d["dram__bytes_write.sum"]) * (1e9 if u["dram__bytes_write.sum"] == "Gbyte" else 1e6 if u["dram__bytes_write.sum"] == "Mbyte" else 1)
            traffic = rd + wr
        except Exception:
            pass
    return "\n".join(lines), traffic


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    agg = {}
    total = 0.0
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(d["Metric Unit"], 1e-9)
        name = d["Kernel Name"].split("(")[0][:90]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
        total += v * scale
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for name, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{name}` | {cnt} | {t*1e3:.3f} | {t/total*100:.2f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        text, traffic = summarise(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
        print(text)
        if traffic is not None:
            print(f"\ntraffic_bytes_per_launch: {traffic:.0f}")
