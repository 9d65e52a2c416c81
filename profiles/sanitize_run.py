"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck): every
algorithm of the C ABI once on small graphs, results checked against the oracle.
usage: compute-sanitizer --tool memcheck python profiles/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
g = simgen.rmat(11, 8, seed=3, wmin=1, wmax=255)
G = ctx.upload(g)
checks = {}


def chk(name, val):
    checks[name] = bool(val)


for kw in ({}, dict(fusion=2), dict(force_dir=1), dict(force_filter=2)):
    chk(f'bfs{kw}', np.array_equal(G.bfs(0, **kw)[0], oracle.bfs(g, 0)))
chk('sssp_d256', np.array_equal(G.sssp(0, 256)[0], oracle.sssp(g, 0)))
chk('sssp_bf', np.array_equal(G.sssp(0, 0, cluster_enter=0)[0], oracle.sssp(g, 0)))
chk('kcore', np.array_equal(G.kcore(0)[0], oracle.coreness(g)))
chk('kcore_bsp', np.array_equal(G.kcore(0, cluster_enter=0)[0], oracle.coreness(g)))
chk('wcc', np.array_equal(G.wcc()[0], oracle.wcc(g)))
r = G.pagerank(0.85, 5)[0]
chk('pagerank', np.max(np.abs(r - oracle.pagerank(g, 0.85, 5)) / oracle.pagerank(g, 0.85, 5)) < 1e-5)
rc, st, _ = G.pagerank_conv(0.85, 1e-8, 100000, 0, force_dir=1)
ref, _, _ = oracle.pagerank_conv(g, 0.85, 1e-12, 100000, 0)
chk('pagerank_conv', np.abs(rc - ref).sum() <= 0.85 / 0.15 * 1.0001e-8 + 1e-12)
pr = simgen.bp_prior(1, g.n)
o, t = oracle.bp(g, pr, 3, with_abs_terms=True)
chk('bp', bool(np.all(np.abs(G.bp(pr, 3)[0] - o) <= 1e-5 * (np.abs(o) + t))))
x = simgen.uniform_f32(1, 1, g.n, 0.0, 1.0)
chk('spmv', np.allclose(G.spmv(x, 1)[0], oracle.spmv(g, x), rtol=1e-5))
lv = torch.empty(g.n, dtype=torch.int32, device="cuda")
G.bfs_async(0, lv)
G.sync()
chk('bfs_async', np.array_equal(lv.cpu().numpy().view(np.uint32), oracle.bfs(g, 0)))
G.free()
D = simdx.Dist(ctx, g.n, 2)
for rnk in range(2):
    lo, hi = D.range(rnk)
    rp = (g.row_ptr[lo:hi + 1] - g.row_ptr[lo]).astype(np.uint64)
    D.upload(rnk, simgen.CSR(n=g.n, row_ptr=rp, col=g.col[g.row_ptr[lo]:g.row_ptr[hi]].copy(),
                             w=g.w[g.row_ptr[lo]:g.row_ptr[hi]].copy(), v_lo=lo, v_hi=hi))
chk('dist_bfs', np.array_equal(np.concatenate(D.bfs(0)[0]), oracle.bfs(g, 0)))
chk('dist_sssp', np.array_equal(np.concatenate(D.sssp(0, 256)[0]), oracle.sssp(g, 0)))
D.free()
ctx.close()
bad = [k for k, v in checks.items() if not v]
print("sanitize_run parity:", "ok" if not bad else f"MISMATCH in {bad}", f"({len(checks)} checks)")
