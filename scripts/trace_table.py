"""Tabulate a DDB_LAPACK_TRACE=1 Rpotrf timeline (the last call in the log):
per outer block J the lookahead update, the diagonal block, the panel, and
the bulk trailing update rest(J-1) running beside them.  trace_table.py log [nb]"""
import sys

lines = [l.split() for l in open(sys.argv[1]) if l.startswith("trace")]
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 256
starts = [i for i, l in enumerate(lines) if l[2] == "panel_done" and l[3] == "0"]
k = starts[-1] - 1
while k >= 0 and lines[k][2] == "diagblk_done":
    k -= 1
ev = {}
for l in lines[k + 1:]:
    ev.setdefault((l[2], int(l[3])), float(l[1]))
f = lambda x: f"{x:8.2f}" if x is not None else "    -   "
J = 0
while ("panel_done", J) in ev:
    g = lambda w, j: ev.get((w, j))
    print(f"J={J:5d} upd {f(g('upd_start', J - nb))}->{f(g('upd_done', J - nb))} "
          f"diagblk {f(g('diagblk_done', J))} panel {f(g('panel_done', J))} | "
          f"rest(J-1) {f(g('rest_start', J - nb))}->{f(g('rest_done', J - nb))}")
    J += nb
