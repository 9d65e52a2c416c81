"""The shared input generator: determinism, CSR invariants,
symmetric weights, relabel bijectivity, Philox known answer."""
import numpy as np

import simgen


def test_philox_known_answer():
    # Random123 philox4x32-10 KAT: counter 0, key 0
    assert simgen.philox(0, 0, 0, 0, 0) == (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)


def test_relabel_bijective_fixes_zero():
    for bits in (1, 5, 10, 16):
        xs = [simgen.relabel(x, bits) for x in range(1 << bits)]
        assert sorted(xs) == list(range(1 << bits))
        assert xs[0] == 0


def _check_csr(g, symmetric=True):
    rp = g.row_ptr
    assert rp[0] == 0 and np.all(np.diff(rp.astype(np.int64)) >= 0) and rp[-1] == g.col.size
    assert g.col.size == 0 or g.col.max() < g.n
    deg = np.diff(rp).astype(np.int64)
    src = np.repeat(np.arange(g.n), deg)
    assert not np.any(src == g.col), "self-loops must be dropped"
    for v in range(min(g.n, 200)):
        row = g.col[rp[v]:rp[v + 1]]
        assert np.all(np.diff(row.astype(np.int64)) >= 0)
    if symmetric:
        w = np.zeros(g.col.size, np.int64) if g.w is None else g.w.astype(np.int64)
        a = np.stack([src, g.col.astype(np.int64), w], 1)
        b = np.stack([g.col.astype(np.int64), src, w], 1)
        a = a[np.lexsort(a.T[::-1])]
        b = b[np.lexsort(b.T[::-1])]
        assert np.array_equal(a, b)


def test_rmat_deterministic_and_valid():
    g1 = simgen.rmat(10, 16, 1, 1, 255)
    g2 = simgen.rmat(10, 16, 1, 1, 255)
    assert np.array_equal(g1.row_ptr, g2.row_ptr) and np.array_equal(g1.col, g2.col)
    assert np.array_equal(g1.w, g2.w)
    _check_csr(g1)
    assert g1.w.min() >= 1 and g1.w.max() <= 255
    deg = g1.degree()
    assert deg[0] == deg.max()  # the relabel fixes the hub at vertex 0
    g3 = simgen.rmat(10, 16, 2)
    assert not np.array_equal(g1.col[:100], g3.col[:100])


def test_rmat_partition_rows_concatenate():
    g = simgen.rmat(9, 8, 3, 1, 255)
    parts = [simgen.rmat(9, 8, 3, 1, 255, v_lo=lo, v_hi=hi) for lo, hi in ((0, 100), (100, 300), (300, 512))]
    col = np.concatenate([p.col for p in parts])
    assert np.array_equal(col, g.col)
    assert np.array_equal(np.concatenate([p.w for p in parts]), g.w)
    deg = np.concatenate([np.diff(p.row_ptr) for p in parts])
    assert np.array_equal(deg, g.degree())


def test_grid():
    g = simgen.grid(5, 7, seed=3)
    _check_csr(g)
    assert g.m == 2 * (5 * 6 + 4 * 7)
    deg = g.degree().reshape(5, 7)
    assert deg[0, 0] == 2 and deg[2, 3] == 4 and deg[0, 3] == 3
    assert g.w.min() >= 1


def test_from_edges_keeps_duplicates_drops_loops():
    g = simgen.from_edges(3, [(0, 1), (0, 1), (2, 2), (1, 2)], [3, 4, 5, 6])
    assert list(g.degree()) == [2, 3, 1]
    assert list(g.col) == [1, 1, 0, 0, 2, 1]
    assert list(g.w) == [3, 4, 3, 4, 6, 6]


def test_directed_has_csc():
    g = simgen.from_edges(3, [(0, 1), (0, 2), (1, 2)], symmetric=False)
    assert list(g.row_ptr) == [0, 2, 3, 3]
    assert list(g.csc_ptr) == [0, 0, 1, 3]
    assert list(g.csc_idx) == [0, 0, 1]


def test_uniform():
    x = simgen.uniform_f32(1, 0, 1000, 0.1, 0.9)
    assert x.min() >= 0.1 and x.max() < 0.9
    assert np.array_equal(x, simgen.uniform_f32(1, 0, 1000, 0.1, 0.9))
