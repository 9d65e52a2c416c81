"""C5-scale parity on one GPU: BASELINE.json config 5, R-MAT scale 27 (134 M
vertices, 4.3 G directed edges, more than 2^32 - 1: u64 edge indices on the
whole path), generated on the device (SX_C5_SCALE overrides the scale).  BFS is compared element by element with the oracle
(queue BFS over the downloaded CSR); SSSP (delta = 1024, the bench setting) is
checked on the device by the properties that define shortest-path distances at
any size: dist(src) = 0, dist(v) <= dist(u) + w(u,v) on every
edge, every reached v != src has a tight in-edge, unreached vertices have no
reached neighbour.  The multi-GPU path at s27 is covered by tests/test_gpu_dist.py
(virtual ranks) and bench.py --gpus N."""
import os

import numpy as np
import pytest

import oracle
import simgen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
INF = 0xFFFFFFFF
SCALE = int(os.environ.get("SX_C5_SCALE", "27"))


@pytest.fixture(scope="module")
def big():
    import torch
    from paper_1812_04070_b200 import simdx
    torch.cuda.set_device(0)
    ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
    G = ctx.rmat(SCALE, 16, 1, 1, 255)
    yield ctx, G
    G.free()
    ctx.close()


def _csr_on_device(G):
    import torch
    from paper_1812_04070_b200 import simdx
    n, m, _, _ = G.info()
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda:0")
    col = torch.empty(m, dtype=torch.int32, device="cuda:0")
    w = torch.empty(m, dtype=torch.int32, device="cuda:0")
    simdx.sx_graph_download(G.h, rp, col, w)
    return n, m, rp, col, w


def test_c5_scale_bfs_matches_oracle(big):
    import torch
    ctx, G = big
    n, m, _, _ = G.info()
    out = torch.empty(n, dtype=torch.int32, device="cuda:0")
    G.bfs(0, out=out)
    rp = np.empty(n + 1, np.uint64)
    col = np.empty(m, np.uint32)
    from paper_1812_04070_b200 import simdx
    simdx.sx_graph_download(G.h, rp, col, None)
    ref = oracle.bfs(simgen.CSR(n=n, row_ptr=rp, col=col), 0)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref)


def test_c5_scale_sssp_shortest_path_properties(big):
    import torch
    ctx, G = big
    n, m, rp, col, w = _csr_on_device(G)
    d32 = torch.empty(n, dtype=torch.int32, device="cuda:0")
    G.sssp(0, 1024, out=d32)
    dist = d32.to(torch.int64) & 0xFFFFFFFF
    inf = 0xFFFFFFFF
    assert int(dist[0]) == 0
    tight = torch.zeros(n, dtype=torch.bool, device="cuda:0")
    reached_nb = torch.zeros(n, dtype=torch.bool, device="cuda:0")
    deg = rp[1:] - rp[:-1]
    step = 1 << 22
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        e0, e1 = int(rp[r0]), int(rp[r1])
        if e1 == e0:
            continue
        src = torch.repeat_interleave(torch.arange(r0, r1, device="cuda:0"), deg[r0:r1])
        dst = col[e0:e1].to(torch.int64) & 0xFFFFFFFF
        we = w[e0:e1].to(torch.int64)
        ds, dd = dist[src], dist[dst]
        ok = (ds == inf) | (dd <= ds + we)  # relaxed everywhere
        assert bool(ok.all()), f"edge not relaxed in rows [{r0}, {r1})"
        t = (ds != inf) & (ds + we == dd)
        tight.index_fill_(0, dst[t], True)
        reached_nb.index_fill_(0, dst[ds != inf], True)
    reached = dist != inf
    reached[0] = False
    assert bool(tight[reached].all()), "a reached vertex has no tight in-edge"
    assert not bool((reached_nb & (dist == inf)).any()), "an unreached vertex has a reached neighbour"
