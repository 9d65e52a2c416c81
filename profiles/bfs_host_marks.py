"""Host-side timeline of sx_bfs calls (SX_TIMING=2 build marks: prologue, enqueue,
sync, end) plus the Python gap between calls.  usage: SX_TIMING=2 python profiles/bfs_host_marks.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
d = simgen.rmat_gpu(24, 16, 1)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
for _ in range(5):
    G.bfs(0, out=out)
prev = None
for _ in range(8):
    t = time.perf_counter()
    if prev is not None:
        print(f"python gap between calls: {(t - prev) * 1e6:.1f} us", file=sys.stderr)
    G.bfs(0, out=out)
    prev = time.perf_counter()
