"""Top SASS instructions by warp-stall samples from an ncu report (source
page), with their neighbourhood: ncu_hot.py report.ncu-rep [top] [context]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
key = "Warp Stall Sampling (All Samples)"
tot = sum(int(d[key] or 0) for d in data)
print(f"samples {tot}, instructions {len(data)}, executed {sum(int(d['Instructions Executed'] or 0) for d in data)}")
order = sorted(range(len(data)), key=lambda i: -int(data[i][key] or 0))[:top]
for i in sorted(order):
    for j in range(max(0, i - ctx), min(len(data), i + ctx + 1)):
        d = data[j]
        mark = ">" if j == i else " "
        print(f"{mark}{j:5d} {int(d[key] or 0):6d} {100*int(d[key] or 0)/max(tot,1):5.1f}% {d['Instructions Executed']:>9} {d['Source'][:90]}")
    if ctx:
        print()
