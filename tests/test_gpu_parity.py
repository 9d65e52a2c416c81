"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element on the same seeded inputs (bit-exact for BFS / SSSP / k-core, the
north_star tolerances for PageRank / SpMV / BP), across the forced modes of the
JIT filter, the direction switch and the fusion."""
import numpy as np
import pytest

import oracle
import simgen

pytestmark = pytest.mark.gpu
INF = 0xFFFFFFFF


@pytest.fixture(scope="module")
def ctx():
    import torch
    from paper_1812_04070_b200 import simdx
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    c = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
    yield c
    c.close()


def up(ctx, g):
    return ctx.upload(g)


# ---------------------------------------------------------------- tiny adversarial graphs
def tiny_graphs():
    gs = {}
    gs["single"] = simgen.from_edges(1, [], [])
    gs["path"] = simgen.from_edges(6, [(i, i + 1) for i in range(5)], [3, 1, 4, 1, 5])
    gs["two_comp"] = simgen.from_edges(7, [(0, 1), (1, 2), (3, 4), (4, 5), (5, 6)], [1, 2, 3, 4, 5])
    gs["loops_dups"] = simgen.from_edges(5, [(0, 0), (0, 1), (0, 1), (1, 2), (2, 2), (2, 3), (3, 4), (3, 4)],
                                         [9, 2, 7, 1, 1, 5, 3, 2])
    gs["clique40"] = simgen.from_edges(40, [(a, b) for a in range(40) for b in range(a + 1, 40)],
                                       [1 + (a * 7 + b) % 255 for a in range(40) for b in range(a + 1, 40)])
    # bin boundaries: hubs of degree exactly 31/32/127/128 chained by a path
    edges, w, base = [], [], 4
    for i, d in enumerate((31, 32, 127, 128)):
        for j in range(d - (1 if i in (0, 3) else 2)):
            edges.append((i, base))
            w.append(1 + j % 200)
            base += 1
    edges += [(0, 1), (1, 2), (2, 3)]
    w += [5, 5, 5]
    gs["bins"] = simgen.from_edges(base, edges, w)
    # star with a hub of degree 100000 (grid-split "huge" class)
    k = 100000
    gs["star"] = simgen.from_edges(k + 1, [(0, i) for i in range(1, k + 1)], [1 + i % 255 for i in range(1, k + 1)])
    return gs


TINY = tiny_graphs()


@pytest.mark.parametrize("name", sorted(TINY))
def test_tiny_bfs_sssp_kcore(ctx, name):
    g = TINY[name]
    G = up(ctx, g)
    try:
        for src in sorted({0, g.n - 1, g.n // 2}):
            lv, _, _ = G.bfs(src)
            assert np.array_equal(lv, oracle.bfs(g, src)), (name, src)
            for delta in (0, 4, 1024):
                d, _, _ = G.sssp(src, delta)
                assert np.array_equal(d, oracle.sssp(g, src)), (name, src, delta)
        core, _, _ = G.kcore(0)
        for kw in (dict(force_dir=2, cluster_enter=0), dict(force_dir=2)):  # pull sub-rounds
            c2, _, _ = G.kcore(0, **kw)
            assert np.array_equal(c2, oracle.coreness(g)), (name, kw)
        assert np.array_equal(core, oracle.coreness(g)), name
        for k in (1, 2, 3, 32):
            m, _, _ = G.kcore(k)
            assert np.array_equal(m, oracle.kcore_mask(g, k)), (name, k)
    finally:
        G.free()


def test_fig1_reconstruction_sssp(ctx):
    g = simgen.from_edges(9, [(0, 1), (0, 3), (1, 2), (2, 3), (3, 4), (2, 5), (4, 5), (4, 6), (4, 7), (4, 8)],
                          [5, 1, 2, 1, 3, 6, 2, 1, 4, 2])
    G = up(ctx, g)
    d, st, tr = G.sssp(0, 0, trace_cap=64)
    assert list(d) == [0, 4, 2, 1, 4, 6, 5, 8, 6]
    assert list(d) == list(oracle.sssp(g, 0))
    G.free()


# ---------------------------------------------------------------- BFS forced modes
MODES = [dict(), dict(force_dir=1), dict(force_dir=2), dict(force_filter=1), dict(force_filter=2),
         dict(fusion=0), dict(overflow_threshold=1), dict(overflow_threshold=1 << 20),
         dict(sep_small=4, sep_large=8, sep_huge=64), dict(force_dir=2, fusion=0),
         dict(cluster_enter=0), dict(cluster_enter=64), dict(cluster_enter=1 << 20),
         dict(fusion=2), dict(fusion=2, force_dir=1), dict(fusion=2, force_dir=2), dict(fusion=2, force_filter=2),
         dict(fusion=2, force_filter=1, overflow_threshold=1),
         dict(force_filter=3), dict(force_filter=3, force_dir=1), dict(fusion=2, force_filter=3)]  # batch


@pytest.fixture(scope="module")
def rmat14():
    return simgen.rmat(14, 16, seed=3, wmin=1, wmax=255)


@pytest.mark.parametrize("mode", MODES, ids=[str(m) for m in MODES])
def test_bfs_modes_rmat(ctx, rmat14, mode):
    G = up(ctx, rmat14)
    ref = oracle.bfs(rmat14, 0)
    for src in (0, 77):
        r = oracle.bfs(rmat14, src) if src else ref
        lv, st, tr = G.bfs(src, trace_cap=256, **mode)
        assert np.array_equal(lv, r), mode
        # per-level frontier sizes = the oracle's level histogram (exact; the batch
        # filter counts its duplicates, so its push levels can only count more)
        hist = oracle.level_histogram(r)
        got = [t["n_frontier"] for t in tr if t["iter"] > 0]  # iteration 0: the fused init record
        if mode.get("force_filter") == 3:
            assert all(g >= h for g, h in zip(got, hist[1:])), (got, hist)
        else:
            assert got[:len(hist) - 1] == list(hist[1:]), (got, hist)
    G.free()


SK_MODES = MODES[:6] + [dict(force_filter=3), dict(force_filter=3, cluster_enter=0), dict(force_dir=2, cluster_enter=0), dict(force_dir=2, fusion=0), dict(local_chain=0), dict(local_chain=100000),
                        dict(local_chain=3, force_filter=2), dict(cluster_enter=0), dict(cluster_enter=1 << 20)]


@pytest.mark.parametrize("ce", [0, 16, 2048, 1 << 20])
def test_cluster_mode_grid_and_star(ctx, ce):
    # small-frontier cluster mode: a grid (long diameter, frontiers in and out of
    # the cluster range) and a star (one task of degree > CL_BIG split cluster-wide)
    g = simgen.grid(96, 80, 5, 1, 255)
    star = simgen.from_edges(3000, [(0, i) for i in range(1, 3000)] + [(i, i + 1) for i in range(1, 2999)],
                             [7] * 2999 + [1] * 2998)
    for gr, srcs in ((g, (0, 4000)), (star, (0, 5))):
        G = up(ctx, gr)
        try:
            for src in srcs:
                lv, st, tr = G.bfs(src, cluster_enter=ce, trace_cap=20000)
                assert np.array_equal(lv, oracle.bfs(gr, src)), (ce, src)
                hist = oracle.level_histogram(lv)
                assert [t["n_frontier"] for t in tr][:len(hist) - 1] == list(hist[1:])
                if ce == 0:
                    assert all(t["dir"] != 2 for t in tr)
                for delta in (0, 3, 600):
                    d, _, tr = G.sssp(src, delta, cluster_enter=ce, trace_cap=20000)
                    assert np.array_equal(d, oracle.sssp(gr, src)), (ce, src, delta)
                    if ce == 0:
                        assert all(t["dir"] != 2 for t in tr)
        finally:
            G.free()


@pytest.mark.parametrize("mode", SK_MODES, ids=[str(m) for m in SK_MODES])
def test_sssp_kcore_modes_rmat(ctx, rmat14, mode):
    G = up(ctx, rmat14)
    for delta in (0, 64, 1024):
        d, st, _ = G.sssp(0, delta, **mode)
        assert np.array_equal(d, oracle.sssp(rmat14, 0)), (mode, delta)
        if mode.get("force_dir") == 2:
            assert st["pull_iters"] > 0
        if mode.get("force_dir") == 1:
            assert st["pull_iters"] == 0
    # k-core takes force_dir too: 2 = pull sub-rounds, 1 = push only
    core, st, _ = G.kcore(0, **mode)
    assert np.array_equal(core, oracle.coreness(rmat14)), mode
    if mode.get("force_dir") == 2 and mode.get("cluster_enter") == 0:
        assert st["pull_iters"] > 0
    if mode.get("force_dir") == 1:
        assert st["pull_iters"] == 0
    mk, _, _ = G.kcore(16, **mode)
    assert np.array_equal(mk, oracle.kcore_mask(rmat14, 16)), mode
    G.free()


# ---------------------------------------------------------------- pull-all (PR / SpMV / BP)
def pr_check(r, o):
    assert np.max(np.abs(r.astype(np.float64) - o) / o) <= 1e-5


@pytest.mark.parametrize("name", ["rmat14", "star", "clique40", "directed"])
def test_pagerank_spmv_bp(ctx, rmat14, name):
    if name == "rmat14":
        g = rmat14
    elif name == "directed":
        g = simgen.random_graph(3000, 20000, 5, wmin=1, wmax=255, symmetric=False)
    else:
        g = TINY[name]
    G = up(ctx, g)
    for T in (1, 20):
        r, st, tr = G.pagerank(0.85, T, trace_cap=64)
        pr_check(r, oracle.pagerank(g, 0.85, T))
        assert tr[0]["filter"] == 1 and all(t["filter"] == 2 for t in tr[1:])  # ballot exactly in iteration 1
    x = simgen.uniform_f32(7, 1, g.n, 0.0, 1.0)
    y, _, _ = G.spmv(x, 3)
    o = oracle.spmv(g, x)
    assert np.all(np.abs(y - o) <= 1e-5 * np.maximum(np.abs(o), 1e-30))
    p = simgen.bp_prior(11, g.n)
    for T in (1, 10):
        l, _, _ = G.bp(p, T)
        o, at = oracle.bp(g, p, T, with_abs_terms=True)
        assert np.all(np.abs(l - o) <= 1e-5 * (np.abs(o) + at)), T
    G.free()


# ---------------------------------------------------------------- errors and edge cases
def test_errors(ctx):
    from paper_1812_04070_b200 import simdx
    g = simgen.from_edges(3, [(0, 1), (1, 2)])
    G = up(ctx, g)
    with pytest.raises(simdx.SimdxError) as e:
        G.bfs(3)
    assert e.value.status == simdx.SX_E_INVALID
    with pytest.raises(simdx.SimdxError) as e:
        G.sssp(0)
    assert e.value.status == simdx.SX_E_WEIGHT
    G.free()
    gz = simgen.from_edges(3, [(0, 1), (1, 2)], [1, 0])
    Gz = up(ctx, gz)
    with pytest.raises(simdx.SimdxError) as e:
        Gz.sssp(0)
    assert e.value.status == simdx.SX_E_WEIGHT
    Gz.free()
    gd = simgen.from_edges(3, [(0, 1), (1, 2)], symmetric=False)
    from paper_1812_04070_b200.simdx import sx_graph_upload, sx_graph_free, Graph
    h = sx_graph_upload(ctx.h, gd.n, gd.row_ptr, gd.col, None, None, None, None, True)
    Gd = Graph(ctx, h, gd.n)
    with pytest.raises(simdx.SimdxError) as e:
        Gd.pagerank()
    assert e.value.status == simdx.SX_E_NO_REVERSE
    with pytest.raises(simdx.SimdxError) as e:
        Gd.kcore(0)
    assert e.value.status == simdx.SX_E_INVALID
    lv, _, _ = Gd.bfs(0, force_dir=1)
    assert list(lv) == [0, 1, 2]
    Gd.free()
    bad = simgen.from_edges(3, [(0, 1)])
    bad.col = bad.col.copy()
    bad.col[0] = 7
    with pytest.raises(simdx.SimdxError) as e:
        up(ctx, bad)
    assert e.value.status == simdx.SX_E_INVALID


@pytest.mark.parametrize("directed", [False, True])
def test_dense_sssp_wcc_cluster_tail(ctx, directed):
    """Dense weighted graphs in the one-cluster tail: without a claim
    every improvement is an append, so an iteration can produce several times n
    entries; the appends are bounded and an overflowing iteration goes back to
    the grid kernels.  K_1200 with random u8 weights, push only, delta 0 and 64."""
    n = 1200
    rng = np.random.default_rng(11)
    edges = [(a, b) for a in range(n) for b in range(a + 1, n)]
    if directed:
        edges += [(b, a) for a, b in edges]
    w = rng.integers(1, 256, len(edges))
    g = simgen.from_edges(n, edges, w, symmetric=not directed)
    G = up(ctx, g)
    try:
        for src in (0, n - 1):
            ref = oracle.sssp(g, src)
            for delta in (0, 64):
                for mode in (dict(force_dir=1, cluster_enter=1 << 20), dict(cluster_enter=1 << 20), dict()):
                    d, _, _ = G.sssp(src, delta, **mode)
                    assert np.array_equal(d, ref), (src, delta, mode)
        if not directed:
            lab, _, _ = G.wcc(force_dir=1, cluster_enter=1 << 20)
            assert np.array_equal(lab, oracle.wcc(g))
    finally:
        G.free()


def test_directed_bfs_sssp_with_csc(ctx):
    g = simgen.random_graph(2000, 12000, 9, wmin=1, wmax=255, symmetric=False)
    G = up(ctx, g)
    for mode in (dict(), dict(force_dir=2), dict(force_dir=1)):
        lv, _, _ = G.bfs(0, **mode)
        assert np.array_equal(lv, oracle.bfs(g, 0)), mode
    d, _, _ = G.sssp(0, 128)
    assert np.array_equal(d, oracle.sssp(g, 0))
    G.free()


def test_device_info(ctx):
    info = ctx.info()
    assert info["sm_count"] >= 100 and info["cc_major"] == 10
    assert info["push_ctas_per_sm"] >= 1 and info["pull_ctas_per_sm"] >= 1
    # Eq. 1 generalised: grid = ctas/SM x SMs fits the register file
    assert info["push_ctas_per_sm"] * info["block_threads"] * info["push_regs"] <= info["regs_per_sm"]


def test_device_pointers_in_and_out(ctx, rmat14):
    import torch
    from paper_1812_04070_b200.simdx import sx_graph_upload, Graph
    dev = torch.device("cuda:0")
    rp = torch.from_numpy(rmat14.row_ptr.view(np.int64)).to(dev)
    ci = torch.from_numpy(rmat14.col.view(np.int32)).to(dev)
    w = torch.from_numpy(rmat14.w).to(dev)
    h = sx_graph_upload(ctx.h, rmat14.n, rp, ci, w, borrow=True)
    G = Graph(ctx, h, rmat14.n)
    out = torch.empty(rmat14.n, dtype=torch.int32, device=dev)
    G.bfs(0, out=out)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), oracle.bfs(rmat14, 0))
    G.free()


def tile_edge_graph(degs, n_src=3000, seed=3, E_extra=0):
    """Directed graph whose in-degrees follow `degs` (cycled), sources uniform: rows
    that end exactly on, straddle and span the pull kernel's 256-edge tiles."""
    rng = np.random.default_rng(seed)
    n = n_src
    edges = []
    for u in range(n):
        d = degs[u % len(degs)]
        for v in rng.integers(0, n, d):
            if v != u:
                edges.append((int(v), u))
    w = [1 + (i * 37) % 255 for i in range(len(edges))]
    return simgen.from_edges(n, edges, w, symmetric=False)


@pytest.mark.parametrize("degs", [[256], [255, 1], [257, 0, 0, 3], [0, 0, 0, 700, 1, 2], [1], [511, 256, 0, 1]])
def test_tiled_pull_row_boundaries(ctx, degs):
    """All-active pull (PageRank / SpMV / BP) on rows that end on, straddle and span the
    256-edge tiles, with empty rows in between (directed: CSC in-rows)."""
    g = tile_edge_graph(degs, n_src=1500 if max(degs) > 300 else 3000)
    G = up(ctx, g)
    r, _, _ = G.pagerank(0.85, 5)
    pr_check(r, oracle.pagerank(g, 0.85, 5))
    x = simgen.uniform_f32(2, 1, g.n, 0.0, 1.0)
    y, _, _ = G.spmv(x, 1)
    o = oracle.spmv(g, x)
    assert np.all(np.abs(y - o) <= 1e-5 * np.maximum(np.abs(o), 1e-30))
    p = simgen.bp_prior(4, g.n)
    l, _, _ = G.bp(p, 3)
    o, at = oracle.bp(g, p, 3, with_abs_terms=True)
    assert np.all(np.abs(l - o) <= 1e-5 * (np.abs(o) + at))
    G.free()


@pytest.mark.parametrize("m", [1, 255, 256, 257, 511, 512, 8192])
def test_tiled_pull_tiny_edge_counts(ctx, m):
    """Edge counts below, on and just past tile multiples (the sentinel row start at E)."""
    rng = np.random.default_rng(m)
    n = 64
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    edges = [(int(a), int(b)) for a, b in zip(src, dst) if a != b]
    g = simgen.from_edges(n, edges, [1 + i % 200 for i in range(len(edges))], symmetric=False)
    G = up(ctx, g)
    r, _, _ = G.pagerank(0.85, 4)
    pr_check(r, oracle.pagerank(g, 0.85, 4))
    G.free()


# ---------------------------------------------------------------- WCC (C-W)
@pytest.mark.parametrize("name", sorted(TINY))
def test_wcc_tiny(ctx, name):
    g = TINY[name]
    G = up(ctx, g)
    lab, _, _ = G.wcc()
    assert np.array_equal(lab, oracle.wcc(g)), name
    G.free()


@pytest.mark.parametrize("mode", SK_MODES, ids=[str(m) for m in SK_MODES])
def test_wcc_modes_rmat(ctx, mode):
    """R-MAT s14 with many small components (ef 2), across the filter / direction / fusion modes."""
    g = simgen.rmat(14, 2, seed=5)
    G = up(ctx, g)
    lab, st, _ = G.wcc(**mode)
    assert np.array_equal(lab, oracle.wcc(g)), mode
    if mode.get("force_dir") == 2:
        assert st["pull_iters"] > 0
    G.free()


def test_wcc_grid_and_generated(ctx):
    """A grid (one component, diameter rows + cols) and the generator's unweighted R-MAT."""
    g = simgen.grid(60, 90, 1, 0, 0)
    G = up(ctx, g)
    lab, _, _ = G.wcc()
    assert not lab.any()
    G.free()
    G = ctx.rmat(13, 4, 7)
    lab, _, _ = G.wcc()
    assert np.array_equal(lab, oracle.wcc(simgen.rmat(13, 4, 7)))
    G.free()


def test_wcc_rejects_directed(ctx):
    from paper_1812_04070_b200 import simdx
    g = simgen.random_graph(100, 300, 2, symmetric=False)
    G = up(ctx, g)
    with pytest.raises(simdx.SimdxError) as e:
        G.wcc()
    assert e.value.status == simdx.SX_E_INVALID
    G.free()


@pytest.mark.parametrize("pos", [0, 7, 8, 1000, -1])
def test_upload_validation_vectorized(ctx, pos):
    """Validation on the 128-bit path (long edge arrays): a column id >= n or a zero weight
    anywhere (head, vector body, scalar tail) is rejected; the clean graph is accepted."""
    from paper_1812_04070_b200 import simdx
    g = simgen.rmat(10, 8, seed=4, wmin=1, wmax=255)
    G = up(ctx, g)  # clean
    G.free()
    bad = simgen.CSR(n=g.n, row_ptr=g.row_ptr, col=g.col.copy(), w=g.w.copy())
    bad.col[pos] = g.n + 5
    with pytest.raises(simdx.SimdxError) as e:
        up(ctx, bad)
    assert e.value.status == simdx.SX_E_INVALID
    zw = simgen.CSR(n=g.n, row_ptr=g.row_ptr, col=g.col, w=g.w.copy())
    zw.w[pos] = 0
    Gz = up(ctx, zw)
    with pytest.raises(simdx.SimdxError) as e:
        Gz.sssp(0)
    assert e.value.status == simdx.SX_E_WEIGHT
    Gz.free()


def test_empty_and_edgeless_graphs(ctx):
    """Degenerate inputs: n = 0 (upload works; BFS/SSSP reject the missing source,
    the source-free algorithms return nothing) and m = 0 (every vertex isolated)."""
    from paper_1812_04070_b200 import simdx
    g0 = simgen.from_edges(0, [])
    G0 = up(ctx, g0)
    with pytest.raises(simdx.SimdxError) as e:
        G0.bfs(0)
    assert e.value.status == simdx.SX_E_INVALID
    for call in (lambda: G0.pagerank(0.85, 3), lambda: G0.kcore(0), lambda: G0.wcc()):
        out, _, _ = call()
        assert out.size == 0
    G0.free()
    n = 1000
    ge = simgen.from_edges(n, [], [])
    Ge = up(ctx, ge)
    lv, _, _ = Ge.bfs(7)
    assert lv[7] == 0 and np.all(np.delete(lv, 7) == INF)
    r, _, _ = Ge.pagerank(0.85, 5)
    pr_check(r, oracle.pagerank(ge, 0.85, 5))
    core, _, _ = Ge.kcore(0)
    assert not core.any()
    lab, _, _ = Ge.wcc()
    assert np.array_equal(lab, np.arange(n, dtype=np.uint32))
    x = simgen.uniform_f32(3, 1, n, 0.0, 1.0)
    y, _, _ = Ge.spmv(x, 1)
    assert not y.any()
    Ge.free()


def test_bfs_repeated_source_start_cache(ctx, rmat14):
    """sx_bfs remembers the start direction of the last (source, options): a repeated
    call enqueues no launch that exits at once; results never depend on it."""
    G = up(ctx, rmat14)
    ref0, ref5 = oracle.bfs(rmat14, 0), oracle.bfs(rmat14, 5)
    lv, st1, _ = G.bfs(0)
    assert np.array_equal(lv, ref0)
    lv, st2, _ = G.bfs(0)
    assert np.array_equal(lv, ref0) and st2["launches"] <= st1["launches"]
    for src, ref in ((5, ref5), (0, ref0), (5, ref5)):
        for kw in ({}, dict(cluster_enter=0), dict(force_dir=1)):
            lv, _, _ = G.bfs(src, **kw)
            assert np.array_equal(lv, ref), (src, kw)
    G.free()
