"""Graph500-style BFS from 64 random roots (degree >= 1) on R-MAT s24: harmonic-mean
GTEPS per option set (device time of each run).  usage: python profiles/bfs_roots.py [scale]"""
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
dg = simgen.rmat_gpu(scale, 16, 1)
G = ctx.upload_device(dg)
rp = torch.empty((1 << scale) + 1, dtype=torch.int64, device="cuda:0")
simdx.sx_graph_download(G.h, rp, None, None)
deg = (rp[1:] - rp[:-1])
cand = torch.nonzero(deg > 0).flatten().cpu().numpy()
roots = np.random.default_rng(1).choice(cand, 64, replace=False)
out = torch.empty(1 << scale, dtype=torch.int32, device="cuda:0")
for name, kw in (("fusion2_all", dict(fusion=2, cluster_enter=0)), ("fusion1_selective+cluster", {}),
                 ("fusion1_no_cluster", dict(cluster_enter=0))):
    g = []
    for r in roots:
        G.bfs(int(r), out=out, **kw)
        _, s, _ = G.bfs(int(r), out=out, **kw)
        mc = int(deg[out != -1].sum().item()) // 2
        g.append(mc / (s["ms"] * 1e-3) / 1e9)
    print(f"{name:28s}: hmean {len(g) / sum(1 / x for x in g):7.1f} GTEPS  min {min(g):7.1f}  max {max(g):7.1f}")
