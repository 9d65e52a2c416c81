"""Beamer alpha / beta sweep for the BFS direction switch (reading 8) on R-MAT s24:
time from the hub (vertex 0) and the harmonic-mean GTEPS over 64 random roots,
all fusion.  usage: python profiles/bfs_ab_sweep.py [scale]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
G = ctx.upload_device(simgen.rmat_gpu(scale, 16, 1))
rp = torch.empty((1 << scale) + 1, dtype=torch.int64, device="cuda:0")
simdx.sx_graph_download(G.h, rp, None, None)
deg = (rp[1:] - rp[:-1])
cand = torch.nonzero(deg > 0).flatten().cpu().numpy()
roots = np.random.default_rng(1).choice(cand, 64, replace=False)
out = torch.empty(1 << scale, dtype=torch.int32, device="cuda:0")
mcs = {}
AB = [tuple(map(int, x.split(","))) for x in sys.argv[2:]] or [(14, 24), (30, 24), (30, 128), (60, 24), (60, 128), (100, 128), (200, 128), (60, 512)]
for alpha, beta in AB:
    kw = dict(fusion=2, cluster_enter=0, alpha=alpha, beta=beta)
    hub = min(G.bfs(0, out=out, **kw)[1]["ms"] for _ in range(4))
    g = []
    for r in roots:
        G.bfs(int(r), out=out, **kw)
        _, s, _ = G.bfs(int(r), out=out, **kw)
        if int(r) not in mcs:
            mcs[int(r)] = int(deg[out != -1].sum().item()) // 2
        g.append(mcs[int(r)] / (s["ms"] * 1e-3) / 1e9)
    print(f"alpha {alpha:3d} beta {beta:5d}: hub {hub * 1e3:6.1f} us   random roots hmean {len(g) / sum(1 / x for x in g):7.1f} GTEPS")
