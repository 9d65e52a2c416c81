"""SX_DEDUP (reading 19 keeps duplicate edges by default): the
upload collapses duplicates to one edge per (row, neighbour) with the minimum
weight, neighbours ascending per row.  Checked against a host deduplication of
the same CSR, and the algorithms against the oracle on the deduplicated graph."""
import numpy as np
import pytest

import oracle
import simgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    from paper_1812_04070_b200 import simdx
    torch.cuda.set_device(0)
    c = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
    yield c
    c.close()


def host_dedup(n, rp, col, w):
    """One edge per (row, neighbour), the minimum weight, neighbours ascending."""
    rows = np.repeat(np.arange(n, dtype=np.uint64), np.diff(rp.astype(np.int64)))
    keys = (rows << np.uint64(32)) | col.astype(np.uint64)
    order = np.lexsort((w, keys))  # by key, then weight: the first of a run is its minimum
    ks, ws = keys[order], w[order]
    head = np.ones(len(ks), bool)
    head[1:] = ks[1:] != ks[:-1]
    uk, uw = ks[head], ws[head]
    cnt = np.bincount((uk >> np.uint64(32)).astype(np.int64), minlength=n)
    rp2 = np.zeros(n + 1, np.uint64)
    rp2[1:] = np.cumsum(cnt)
    return rp2, (uk & np.uint64(0xFFFFFFFF)).astype(np.uint32), uw


def test_upload_dedup_rmat(ctx):
    g = simgen.rmat(12, 16, seed=5, wmin=1, wmax=255)  # R-MAT keeps duplicate tuples
    rp2, col2, w2 = host_dedup(g.n, g.row_ptr, g.col, g.w)
    assert len(col2) < len(g.col), "the fixture must contain duplicates"
    G = ctx.upload(g, dedup=True)
    drp, dcol, dw = G.download()
    assert np.array_equal(drp, rp2) and np.array_equal(dcol, col2) and np.array_equal(dw, w2.astype(np.uint32))
    g2 = simgen.CSR(n=g.n, row_ptr=rp2, col=col2, w=w2.astype(g.w.dtype))
    assert np.array_equal(G.bfs(0)[0], oracle.bfs(g2, 0))
    d, _, _ = G.sssp(0, 256)
    assert np.array_equal(d, oracle.sssp(g2, 0))
    assert np.array_equal(d, oracle.sssp(g, 0))  # the minimum weight keeps every shortest path
    assert np.array_equal(G.kcore(0)[0], oracle.coreness(g2))
    r = G.pagerank(0.85, 10)[0]
    o = oracle.pagerank(g2, 0.85, 10)
    assert np.max(np.abs(r - o) / o) <= 1e-5
    G.free()


def test_upload_dedup_directed_and_unweighted(ctx):
    src, dst, w = simgen.rmat_tuples(10, 8, 2, 1, 255)
    g = simgen.csr_from_tuples(1 << 10, src, dst, w, False)  # directed, with its CSC
    rp2, col2, w2 = host_dedup(g.n, g.row_ptr, g.col, g.w)
    crp2, ccol2, cw2 = host_dedup(g.n, g.csc_ptr, g.csc_idx, g.csc_w)
    G = ctx.upload(g, dedup=True)
    drp, dcol, dw = G.download()
    assert np.array_equal(drp, rp2) and np.array_equal(dcol, col2) and np.array_equal(dw, w2.astype(np.uint32))
    g2 = simgen.CSR(n=g.n, row_ptr=rp2, col=col2, w=w2.astype(g.w.dtype), directed=True,
                    csc_ptr=crp2, csc_idx=ccol2, csc_w=cw2.astype(g.csc_w.dtype))
    assert np.array_equal(G.bfs(0)[0], oracle.bfs(g2, 0))
    assert np.array_equal(G.sssp(0, 0)[0], oracle.sssp(g2, 0))
    G.free()
    u = simgen.CSR(n=g.n, row_ptr=g.row_ptr, col=g.col)  # unweighted (and treated as symmetric rows)
    Gu = ctx.upload(u, dedup=True)
    urp, ucol, _ = Gu.download(weights=False)
    assert np.array_equal(urp, rp2) and np.array_equal(ucol, col2)
    Gu.free()
