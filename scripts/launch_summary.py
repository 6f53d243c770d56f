"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel:
count, total, share.  Usage: launch_summary.py launches.csv [first_id]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if int(d["ID"]) < first:
        continue
    name = d["Kernel Name"].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
unit = data[0]["Metric Unit"] if data else "?"
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:6d} {v[1] / 1e3:10.1f} us {100 * v[1] / tot:6.1f}%  {k}")
print(f"launches {sum(v[0] for v in agg.values())}  total {tot / 1e3:.1f} us ({unit} in csv)")
