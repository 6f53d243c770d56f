import sys, torch
sys.path.insert(0, ".")
from paper_2109_13406_b200 import DeviceMatrix, Rsyrk, Rgemm, flop_count
from paper_2109_13406_b200.synth import hashed_dd_device
n, k = int(sys.argv[1]), int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
A = DeviceMatrix(n, k, "dd", n, store=hashed_dd_device(n, k, 0, 1, "cuda"))
C = DeviceMatrix(n, n, "dd", n, store=hashed_dd_device(n, n, 0, 3, "cuda"))
best = 1e9
for it in range(reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); Rsyrk("L", "N", n, k, -1.0, A, n, 1.0, C, n); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 1e3)
f = flop_count("Rsyrk", n, k=n)
macs = n * (n + 1) * k / 2
print(f"syrk L N n={n} k={k}: {best*1e3:.3f} ms  {macs/best/1e9:.1f} G MAC/s  = {7.5*macs/best/18.5e12*100:.1f}% of the FP64 pipe at 7.5/MAC")
