"""Does a degree-ordered vertex numbering speed up the all-active pull (C3)?
Builds R-MAT s22 on the host, relabels vertices by descending degree (hubs
first, so the most-gathered values share cache lines), uploads both graphs and
times sx_pagerank (20 iterations) on each.  usage: python profiles/pr_relabel_probe.py [scale]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
t = time.time()
g = simgen.rmat(scale, 16, 1)
n = g.n
deg = np.diff(g.row_ptr).astype(np.int64)
order = np.argsort(-deg, kind="stable")          # new id -> old id
newid = np.empty(n, np.int64)
newid[order] = np.arange(n)                       # old id -> new id
src = np.repeat(np.arange(n), deg)
s2, d2 = newid[src], newid[g.col.astype(np.int64)]
idx = np.lexsort((d2, s2))
s2, d2 = s2[idx], d2[idx]
rp = np.zeros(n + 1, np.uint64)
np.cumsum(np.bincount(s2, minlength=n), out=rp[1:])
col = d2.astype(np.uint32)
print(f"relabelled in {time.time() - t:.1f}s", flush=True)
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
out = torch.empty(n, dtype=torch.float32, device="cuda:0")
for name, (R, C) in (("original", (g.row_ptr, g.col)), ("degree-ordered", (rp, col))):
    G = simdx.Graph(ctx, simdx.sx_graph_upload(ctx.h, n, R, C), n)
    G.pagerank(0.85, 20, out=out)
    ms = min(G.pagerank(0.85, 20, out=out)[1]["ms"] for _ in range(3))
    r = out.cpu().numpy()
    print(f"{name:15s}: pagerank s{scale} x20 {ms:.3f} ms  (sum {r.sum():.6f})")
    G.free()
