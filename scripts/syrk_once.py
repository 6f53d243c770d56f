import sys; sys.path.insert(0, ".")
import bench, torch
st = torch.cuda.current_stream()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
print(bench._rsyrk(n, n, "fast", torch.device("cuda", 0), st, 1))
