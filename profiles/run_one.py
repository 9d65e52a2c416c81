"""Run one algorithm call on one config (for ncu captures).

usage: python profiles/run_one.py {bfs24|bfs24all|sssp_grid|pr22|kcore24|sssp24} [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

what = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
if what == "sssp_grid":
    g = simgen.grid(2048, 2048, 1, 1, 255)
elif what == "pr22":
    g = simgen.rmat(22, 16, 1)
else:
    g = simgen.rmat(24, 16, 1, wmin=1, wmax=255)
G = ctx.upload(g)
out = torch.empty(g.n, dtype=torch.int32, device="cuda:0")
for _ in range(reps):
    if what == "bfs24":
        _, st, _ = G.bfs(0, out=out)
    elif what == "bfs24all":
        _, st, _ = G.bfs(0, out=out, fusion=2, cluster_enter=0)
    elif what == "sssp_grid":
        _, st, _ = G.sssp(0, 1024, out=out)
    elif what == "sssp24":
        _, st, _ = G.sssp(0, 1024, out=out)
    elif what == "pr22":
        _, st, _ = G.pagerank(0.85, 20, out=out.view(torch.float32))
    elif what == "kcore24":
        _, st, _ = G.kcore(0, out=out)
print(what, st)
G.free()
ctx.close()
