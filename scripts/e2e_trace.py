"""Dev tool: the pipelined host-buffer Rgemm (bench.py's e2e leg) with the
C-ABI's stage trace on.  python scripts/e2e_trace.py [n] [mode]"""
import os
import sys

os.environ.setdefault("DDB_HOST_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
print(bench._e2e(n, n, mode, False, 1, 0, torch.device("cuda", 0)), flush=True)
