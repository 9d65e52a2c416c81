"""sx_bfs_async / sx_graph_sync (all fusion enqueued without a host sync,
P:742-743) against the oracle, and the grid-barrier fault injection
(P:707-711)."""
import numpy as np
import pytest

import oracle
import simgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    from paper_1812_04070_b200 import simdx
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    c = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
    yield c
    c.close()


@pytest.fixture(scope="module")
def rmat14():
    return simgen.rmat(14, 16, seed=3, wmin=1, wmax=255)


@pytest.mark.parametrize("kw", [{}, dict(force_dir=1), dict(force_dir=2), dict(force_filter=2),
                                dict(force_filter=1, overflow_threshold=1)], ids=str)
def test_async_bfs_many_sources(ctx, rmat14, kw):
    """70 runs enqueued back to back (more than the 64-entry event ring), each
    into its own device buffer; every level array equals the oracle's."""
    import torch
    G = ctx.upload(rmat14)
    n = rmat14.n
    srcs = [0, 1, 5, 77, 1000, n - 1] * 12 if not kw else [0, 77, n - 1]
    outs = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in srcs]
    for s, o in zip(srcs, outs):
        G.bfs_async(s, o, **kw)
    st = G.sync()
    assert st["runs"] == len(srcs) and st["launches_fused"] == len(srcs)
    assert st["ms"] > 0 and 0 < st["ms_fused"] <= st["ms"]
    refs = {s: oracle.bfs(rmat14, s) for s in set(srcs)}
    for s, o in zip(srcs, outs):
        assert np.array_equal(o.cpu().numpy().view(np.uint32), refs[s]), (s, kw)
    # the summed counters equal those of the same runs made synchronously (fusion = 2)
    tot = dict(edges_examined=0, iterations=0, pull_iters=0)
    for s in srcs:
        _, s1, _ = G.bfs(s, fusion=2, cluster_enter=0, **kw)
        for k in tot:
            tot[k] += s1[k]
    for k in tot:
        assert st[k] == tot[k], (k, st[k], tot[k])
    assert G.sync()["runs"] == 0  # reset by the previous sync
    G.free()


def test_async_bfs_tiny_and_directed(ctx):
    import torch
    gs = [simgen.from_edges(1, [], []), simgen.from_edges(6, [(i, i + 1) for i in range(5)], [1] * 5),
          simgen.from_edges(7, [(0, 1), (1, 2), (3, 4), (4, 5), (5, 6)], [1] * 5),
          simgen.from_edges(100001, [(0, i) for i in range(1, 100001)], [1] * 100000)]
    for g in gs:
        G = ctx.upload(g)
        o = torch.empty(g.n, dtype=torch.int32, device="cuda")
        for src in sorted({0, g.n - 1}):
            G.bfs_async(src, o)
            G.sync()
            assert np.array_equal(o.cpu().numpy().view(np.uint32), oracle.bfs(g, src))
        G.free()
    d = simgen.random_graph(2000, 12000, 9, symmetric=False)
    G = ctx.upload(d)
    o = torch.empty(d.n, dtype=torch.int32, device="cuda")
    G.bfs_async(0, o)
    G.sync()
    assert np.array_equal(o.cpu().numpy().view(np.uint32), oracle.bfs(d, 0))
    G.free()


def test_async_bfs_rejects_host_output_and_bad_source(ctx, rmat14):
    from paper_1812_04070_b200 import simdx
    import torch
    G = ctx.upload(rmat14)
    with pytest.raises(ValueError):
        G.bfs_async(0, np.empty(rmat14.n, np.uint32))
    o = torch.empty(rmat14.n, dtype=torch.int32, device="cuda")
    with pytest.raises(simdx.SimdxError) as e:
        G.bfs_async(rmat14.n, o)
    assert e.value.status == simdx.SX_E_INVALID
    G.free()


def test_barrier_fault_injection(ctx, rmat14):
    """One CTA more than can be co-resident: the cooperative launch is refused
    (SX_E_BARRIER); a CTA that never arrives: the watchdog fires (SX_E_BARRIER),
    the kernel ends, and the context keeps working."""
    from paper_1812_04070_b200 import simdx
    assert simdx.sx_barrier_fault(ctx.h, 1) == simdx.SX_E_BARRIER
    assert simdx.sx_barrier_fault(ctx.h, 2, 200) == simdx.SX_E_BARRIER
    assert simdx.sx_barrier_fault(ctx.h, 3) == simdx.SX_E_INVALID
    # the context is not poisoned and the watchdog is back at its default
    us, _ = simdx.sx_barrier_bench(ctx.h, 100)
    assert us > 0
    G = ctx.upload(rmat14)
    lv, _, _ = G.bfs(0)
    assert np.array_equal(lv, oracle.bfs(rmat14, 0))
    G.free()
