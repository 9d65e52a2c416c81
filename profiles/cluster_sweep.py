"""BFS from vertex 0 with and without the small-frontier cluster tail across
R-MAT scales (device time, median of 5).  usage: python profiles/cluster_sweep.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
for scale in (14, 16, 18, 20, 22, 24):
    d = simgen.rmat_gpu(scale, 16, 1)
    G = ctx.upload_device(d)
    out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
    row = []
    for ce in (0, 1024, 4096, 16384):
        G.bfs(0, out=out, cluster_enter=ce)
        ts = [G.bfs(0, out=out, cluster_enter=ce)[1]["ms"] for _ in range(5)]
        row.append(f"ce={ce}: {statistics.median(ts) * 1e3:7.1f} us")
    print(f"s{scale}: " + "  ".join(row), flush=True)
    G.free()
    d.free()
ctx.close()
