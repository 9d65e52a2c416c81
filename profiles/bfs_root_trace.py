"""Per-level trace of BFS from a few random roots on R-MAT s24 with and without the
cluster tail (iteration, direction, |F'|, launch index, time since the previous record).
usage: python profiles/bfs_root_trace.py [scale] [nroots]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
G = ctx.upload_device(simgen.rmat_gpu(scale, 16, 1))
rp = torch.empty((1 << scale) + 1, dtype=torch.int64, device="cuda:0")
simdx.sx_graph_download(G.h, rp, None, None)
deg = (rp[1:] - rp[:-1])
cand = torch.nonzero(deg > 0).flatten().cpu().numpy()
roots = np.random.default_rng(1).choice(cand, nroots, replace=False)
out = torch.empty(1 << scale, dtype=torch.int32, device="cuda:0")
names = {0: "push", 1: "pull", 2: "clus"}
for r in roots:
    for kw in ({}, dict(cluster_enter=0)):
        G.bfs(int(r), out=out, **kw)
        _, s, tr = G.bfs(int(r), out=out, trace_cap=128, **kw)
        t0 = tr[0]["t_ns"] if tr else 0
        recs = []
        prev = t0
        for t in tr:
            recs.append(f"it{t['iter']}:{names.get(t['dir'], t['dir'])}:F{t['n_frontier']}:L{t['launch']}:{(t['t_ns'] - prev) / 1e3:.1f}")
            prev = t["t_ns"]
        print(f"root {r} deg {int(deg[r])} {kw}: ms {s['ms']:.3f} launches {s['launches']} | " + " ".join(recs))
