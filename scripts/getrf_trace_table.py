"""Tabulate a DDB_LAPACK_TRACE=1 Rgetrf timeline (the last call in the log):
per outer block J the lookahead update, the four inner panels / applies and
the bulk update rest(J-1) beside them.  getrf_trace_table.py log [step]"""
import sys

lines = [l.split() for l in open(sys.argv[1]) if l.startswith("trace")]
step = int(sys.argv[2]) if len(sys.argv) > 2 else 512
idx = [i for i, l in enumerate(lines) if l[2] == "panel_done" and l[3] == "0"]
k = idx[-1]
while k > 0 and lines[k - 1][2] in ("ipanel_done", "iapply_done"):
    k -= 1
ev = {}
for l in lines[k:]:
    ev.setdefault((l[2], int(l[3])), float(l[1]))
f = lambda x: f"{x:8.2f}" if x is not None else "    -   "
for J in range(0, 1 << 20, step):
    g = lambda w, j: ev.get((w, j))
    if g("ipanel_done", J) is None:
        break
    ip = [g("ipanel_done", J + 64 * i) for i in range(4)]
    ia = [g("iapply_done", J + 64 * i) for i in range(4)]
    print(f"J={J:5d} upd {f(g('upd_start', J - 256))}->{f(g('upd_done', J - 256))} ipanel/iapply "
          + " ".join(f(a) + "/" + f(b) for a, b in zip(ip, ia))
          + f" | rest {f(g('rest_start', J - 256))}->{f(g('rest_done', J - 256))}")
