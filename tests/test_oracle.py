"""Pins for the oracle (-m "not gpu"): the oracle is checked against what the
paper and the mathematics fix — the paper's worked examples, closed forms,
invariants, brute force and independent library routines on tiny inputs —
never against itself or the CUDA path."""
import math
import os

import numpy as np
import pytest

import oracle
import simgen
from oracle import acc_model
import brute

INF = oracle.INF
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load_fig1():
    n, src, edges, facts = None, None, [], []
    for line in open(os.path.join(GOLD, "fig1_sssp.txt")):
        line = line.split("#")[0].strip() if not line.startswith("fact") else line.strip()
        if not line:
            continue
        t = line.split()
        if t[0] == "n":
            n = int(t[1])
        elif t[0] == "src":
            src = int(t[1])
        elif t[0] == "e":
            edges.append((int(t[1]), int(t[2]), int(t[3])))
        elif t[0] == "fact":
            facts.append((int(t[1]), t[2], t[3]))
    return n, src, edges, facts


def fig1_graph():
    n, src, edges, facts = load_fig1()
    g = simgen.from_edges(n, [(a, b) for a, b, _ in edges], [w for _, _, w in edges])
    return g, src, facts


NAMES = "abcdefghi"


def _ids(s):
    return sorted(NAMES.index(x) for x in s.split(","))


# ---------------------------------------------------------------- Fig. 1 / Fig. 6
def test_fig1_text_facts_hold_on_reconstruction():
    g, src, facts = fig1_graph()
    meta, trace = acc_model.run(g, src, "sssp")
    assert len(trace) == 4  # iteration 4 updates nothing: "until no vertex gets updated"
    assert trace[-1]["ballot"] == []
    for it, kind, val in facts:
        rec = trace[it - 1]
        if kind == "meta":
            for kv in val.split(","):
                k, v = kv.split("=")
                assert rec["meta"][NAMES.index(k)] == int(v), (it, kv)
        elif kind == "updated":
            assert rec["bits"][NAMES.index(val)] == "1", (it, val)
        elif kind == "active_set":
            assert sorted(rec["active"]) == _ids(val)
        elif kind == "online_set":
            assert sorted(set(rec["online"])) == _ids(val)
        elif kind == "batch_multiset":
            assert sorted(rec["batch"]) == _ids(val)
        elif kind == "ballot_list":
            assert rec["ballot"] == _ids(val)  # sorted AND unique
        elif kind == "ballot_bits_ad":
            assert rec["bits"][:4] == val
        elif kind == "updates_from":
            # reading 2: "computes two/four neighbors" = neighbours that receive an update
            want = {NAMES.index(k): int(v) for k, v in (x.split("=") for x in val.split(","))}
            prev = trace[it - 2]["meta"]
            got = {}
            cur = list(prev)
            for v in rec["active"]:
                c = 0
                for e in range(int(g.row_ptr[v]), int(g.row_ptr[v + 1])):
                    u, w = int(g.col[e]), int(g.w[e])
                    if cur[v] + w < cur[u]:
                        cur[u] = cur[v] + w
                        c += 1
                got[v] = c
            assert got == want
        else:
            raise AssertionError(kind)
    # b is updated ONLY in iterations 1 and 3
    assert [r["bits"][1] for r in trace] == ["1", "0", "1", "0"]


def test_fig1_oracle_dijkstra_matches_acc_fixpoint_and_floyd():
    g, src, _ = fig1_graph()
    meta, _ = acc_model.run(g, src, "sssp")
    d = oracle.sssp(g, src)
    assert list(d) == meta
    s, t, w = brute.tuples_of(g)
    assert np.array_equal(d, brute.floyd_warshall(g.n, s, t, w, src))


def test_eq1_worked_example():
    kv = dict(l.split() for l in open(os.path.join(GOLD, "eq1.txt")) if l.strip() and not l.startswith("#"))
    got = acc_model.eq1_ctas(int(kv["regs_per_smx"]), int(kv["regs_per_thread"]), int(kv["threads_per_cta"]),
                             int(kv["smx"]))
    assert got == int(kv["ctas"]) == 60


def test_classify_boundaries():
    # P:659 separators 32 / 128; ownership small < 32 <= medium < 128 <= large (reading 17)
    assert acc_model.classify(0) == "small"
    assert acc_model.classify(31) == "small"
    assert acc_model.classify(32) == "medium"
    assert acc_model.classify(127) == "medium"
    assert acc_model.classify(128) == "large"


# ---------------------------------------------------------------- BFS (C-B)
def test_bfs_path_and_components():
    g = simgen.from_edges(5, [(0, 1), (1, 2), (2, 3), (3, 4)])
    assert list(oracle.bfs(g, 0)) == [0, 1, 2, 3, 4]
    g = simgen.from_edges(6, [(0, 1), (1, 2), (3, 4), (4, 5)])
    assert list(oracle.bfs(g, 0)) == [0, 1, 2, INF, INF, INF]
    g = simgen.from_edges(1, [])
    assert list(oracle.bfs(g, 0)) == [0]


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("symmetric", [True, False])
def test_bfs_vs_scipy(seed, symmetric):
    g = simgen.random_graph(40, 60, seed, symmetric=symmetric)
    s, t, _ = brute.tuples_of(g)
    assert np.array_equal(oracle.bfs(g, 0), brute.bfs_levels_scipy(g.n, s, t, 0))


def test_bfs_invariants_rmat():
    g = simgen.rmat(10)
    lv = oracle.bfs(g, 0).astype(np.int64)
    s, t, _ = brute.tuples_of(g)
    reached = lv != INF
    both = reached[s] & reached[t]
    assert np.all(np.abs(lv[s][both] - lv[t][both]) <= 1)
    # level(v) = 1 + min over in-neighbours; unreached iff no reached in-neighbour
    best = np.full(g.n, np.iinfo(np.int64).max)
    np.minimum.at(best, t[reached[s]], lv[s][reached[s]])
    for v in range(g.n):
        if v == 0:
            assert lv[v] == 0
        elif reached[v]:
            assert lv[v] == best[v] + 1
        else:
            assert best[v] == np.iinfo(np.int64).max
    h = oracle.level_histogram(oracle.bfs(g, 0))
    assert h.sum() == reached.sum() and h[0] == 1


# ---------------------------------------------------------------- SSSP (C-S)
@pytest.mark.parametrize("seed", range(12))
def test_sssp_vs_floyd_warshall(seed):
    n = 8 + 4 * seed
    g = simgen.random_graph(n, 2 * n, seed, wmin=1, wmax=255, symmetric=(seed % 2 == 0))
    s, t, w = brute.tuples_of(g)
    for src in (0, n // 2):
        assert np.array_equal(oracle.sssp(g, src), brute.floyd_warshall(n, s, t, w, src))


def test_sssp_vs_scipy_dijkstra_larger():
    g = simgen.random_graph(600, 3000, 7, wmin=1, wmax=300)  # u32 weights path
    assert g.w.dtype == np.uint32
    s, t, w = brute.tuples_of(g)
    assert np.array_equal(oracle.sssp(g, 3), brute.dijkstra_scipy(g.n, s, t, w, 3))


def test_sssp_grid_closed_form_unit_weights():
    L = 37
    g = simgen.grid(L, L, wmin=1, wmax=1)
    d = oracle.sssp(g, 0).reshape(L, L)
    r, c = np.indices((L, L))
    assert np.array_equal(d, (r + c).astype(np.uint32))


def test_sssp_unit_weights_equals_bfs():
    g = simgen.rmat(10, wmin=1, wmax=1)
    assert np.array_equal(oracle.sssp(g, 0), oracle.bfs(g, 0))


def test_sssp_fixpoint_invariants():
    g = simgen.rmat(9, wmin=1, wmax=255)
    d = oracle.sssp(g, 0).astype(np.int64)
    s, t, w = brute.tuples_of(g)
    r = d[s] != INF
    assert np.all(d[t][r] <= d[s][r] + w[r])
    tight = np.zeros(g.n, bool)
    tight[t[r & (d[t] == d[s] + w)]] = True
    reached = d != INF
    reached[0] = False
    assert np.all(tight[reached])


def test_sssp_rejects_zero_weight():
    g = simgen.from_edges(3, [(0, 1), (1, 2)], [1, 0])
    with pytest.raises(ValueError):
        oracle.sssp(g, 0)


# ---------------------------------------------------------------- k-core (C-K)
@pytest.mark.parametrize("seed", range(12))
def test_coreness_vs_exhaustive_peeling(seed):
    g = simgen.random_graph(30, 30 + 10 * seed, seed)
    s, t, _ = brute.tuples_of(g)
    assert np.array_equal(oracle.coreness(g), brute.coreness_by_peeling(g.n, s, t))
    for k in (1, 2, 3, 5):
        assert np.array_equal(oracle.kcore_mask(g, k).astype(bool), brute.peel(g.n, s, t, k))


def test_coreness_closed_forms():
    n = 7
    kn = simgen.from_edges(n, [(a, b) for a in range(n) for b in range(a + 1, n)])
    assert list(oracle.coreness(kn)) == [n - 1] * n
    cyc = simgen.from_edges(6, [(i, (i + 1) % 6) for i in range(6)])
    assert list(oracle.coreness(cyc)) == [2] * 6
    star = simgen.from_edges(6, [(0, i) for i in range(1, 6)])
    assert list(oracle.coreness(star)) == [1] * 6
    iso = simgen.from_edges(4, [(0, 1)])
    assert list(oracle.coreness(iso)) == [1, 1, 0, 0]
    tri = simgen.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    assert list(oracle.kcore_mask(tri, 2)) == [1, 1, 1]
    assert list(oracle.kcore_mask(star, 2)) == [0] * 6
    # duplicates count (multigraph, reading 19): a doubled edge is a 2-core
    dbl = simgen.from_edges(2, [(0, 1), (0, 1)])
    assert list(oracle.coreness(dbl)) == [2, 2]


def test_coreness_invariants_rmat():
    g = simgen.rmat(10)
    core = oracle.coreness(g).astype(np.int64)
    s, t, _ = brute.tuples_of(g)
    deg = g.degree().astype(np.int64)
    assert np.all(core <= deg)
    cnt = np.zeros(g.n, np.int64)
    np.add.at(cnt, s, (core[t] >= core[s]).astype(np.int64))
    assert np.all(cnt >= core)  # each v has >= core(v) neighbours with core >= core(v)


# ---------------------------------------------------------------- PageRank (C-P)
def test_pagerank_converges_to_google_matrix_eigenvector():
    for seed, sym in ((1, True), (2, False), (3, True)):
        g = simgen.random_graph(25, 40, seed, symmetric=sym)
        s, t, _ = brute.tuples_of(g)
        ref = brute.pagerank_eigvec(g.n, s, t, 0.85)
        r = oracle.pagerank(g, 0.85, 300)
        assert np.max(np.abs(r - ref) / ref) < 1e-9


def test_pagerank_mass_conservation_with_dangling():
    g = simgen.rmat(10)
    assert (g.degree() == 0).any()
    for T in (1, 5, 20):
        assert abs(oracle.pagerank(g, 0.85, T).sum() - 1.0) < 1e-12


def test_pagerank_uniform_closed_forms():
    n = 6
    kn = simgen.from_edges(n, [(a, b) for a in range(n) for b in range(a + 1, n)])
    cyc = simgen.from_edges(n, [(i, (i + 1) % n) for i in range(n)], symmetric=False)
    empty = simgen.from_edges(n, [])
    for g in (kn, cyc, empty):
        assert np.allclose(oracle.pagerank(g, 0.85, 20), 1.0 / n, rtol=0, atol=1e-15)
    two = simgen.from_edges(2, [(0, 1)])
    r = oracle.pagerank(two, 0.85, 20)
    assert r[0] == r[1]


def test_pagerank_star_recurrence():
    k, d, T = 9, 0.85, 20
    N = k + 1
    g = simgen.from_edges(N, [(0, i) for i in range(1, N)])
    c, l = 1.0 / N, 1.0 / N
    for _ in range(T):
        c, l = (1 - d) / N + d * k * l, (1 - d) / N + d * c / k
    r = oracle.pagerank(g, d, T)
    assert abs(r[0] - c) < 1e-15 and np.allclose(r[1:], l, rtol=0, atol=1e-15)
    # fixed point c* = (1 + d k) / (N (1 + d))
    r = oracle.pagerank(g, d, 400)
    assert abs(r[0] - (1 + d * k) / (N * (1 + d))) < 1e-14


# ---------------------------------------------------------------- PageRank to convergence (C-PC)
# Both recurrences are contractions of factor d in L1 (column-(sub)stochastic
# transition matrix), so a Jacobi iterate whose last L1 change is delta lies
# within d/(1-d) * delta of the exact fixed point ("till all vertices
# have stable rank values"; "converged when L1 delta < epsilon").
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("eps", [1e-4, 1e-8])
def test_pagerank_conv_within_contraction_bound_of_linear_solve(variant, eps):
    d = 0.85
    for seed, sym in ((1, True), (2, False), (3, True), (4, False)):
        g = simgen.random_graph(30, 50, seed, symmetric=sym)
        s, t, _ = brute.tuples_of(g)
        ref = brute.pagerank_linear_solve(g.n, s, t, d, variant)
        r, it, delta = oracle.pagerank_conv(g, d, eps, 10000, variant)
        assert delta < eps and it >= 1
        assert np.abs(r - ref).sum() <= d / (1 - d) * delta + 1e-12, (seed, variant)


def test_pagerank_conv_stops_at_first_step_below_eps():
    # variant 0 is the fixed-T oracle's recurrence: step `it` is the first whose L1 change is < eps
    g = simgen.rmat(9)
    eps = 1e-7
    r, it, delta = oracle.pagerank_conv(g, 0.85, eps, 10000, 0)
    assert np.array_equal(r, oracle.pagerank(g, 0.85, it))
    prev = np.abs(oracle.pagerank(g, 0.85, it - 1) - oracle.pagerank(g, 0.85, it - 2)).sum()
    assert prev >= eps and delta < eps
    assert abs(r.sum() - 1.0) < 1e-12  # mass conservation (dangling redistributed)


def test_pagerank_conv_spec_examples_and_closed_forms():
    d = 0.85
    one = simgen.from_edges(1, [])
    r, _, _ = oracle.pagerank_conv(one, d, 1e-12, 100, 1)
    assert abs(r[0] - 0.15) < 1e-15  # S:489 single vertex -> 1 - d
    two = simgen.from_edges(2, [(0, 1)])
    for v in (0, 1):
        r, _, _ = oracle.pagerank_conv(two, d, 1e-12, 1000, v)
        assert r[0] == r[1]  # S:488 symmetry
    # directed cycle: every vertex has one in- and one out-edge; the fixed point is the start
    cyc = simgen.from_edges(7, [(i, (i + 1) % 7) for i in range(7)], symmetric=False)
    r, it, delta = oracle.pagerank_conv(cyc, d, 1e-12, 100, 1)
    assert it == 1 and delta == 0.0 and np.all(r == 1.0)
    # star K_{1,k}: normalised c* = (1 + d k) / (N (1 + d)); SPEC variant c* = (1 + d k) / (1 + d)
    k = 9
    N = k + 1
    star = simgen.from_edges(N, [(0, i) for i in range(1, N)])
    r, _, delta = oracle.pagerank_conv(star, d, 1e-13, 10000, 0)
    assert abs(r[0] - (1 + d * k) / (N * (1 + d))) < 1e-12
    r, _, delta = oracle.pagerank_conv(star, d, 1e-13, 10000, 1)
    c = (1 + d * k) / (1 + d)
    assert abs(r[0] - c) < 1e-12 and np.allclose(r[1:], (1 - d) + d * c / k, rtol=0, atol=1e-12)
    # SPEC invariant: every rank >= 1 - d (the empty sum is the minimum)
    g = simgen.random_graph(500, 3000, 7, symmetric=False)
    r, _, _ = oracle.pagerank_conv(g, d, 1e-9, 10000, 1)
    assert r.min() >= 1 - d - 1e-15
    # random G(500, 3000) against dense power iteration within 1e-6 L1
    s, t, _ = brute.tuples_of(g)
    assert np.abs(r - brute.pagerank_linear_solve(g.n, s, t, d, 1)).sum() < 1e-6


# ---------------------------------------------------------------- SpMV (C-V)
@pytest.mark.parametrize("sym", [True, False])
def test_spmv_vs_dense_matvec(sym):
    g = simgen.random_graph(50, 200, 5, wmin=1, wmax=255, symmetric=sym)
    x = simgen.uniform_f32(3, 1, g.n, -1.0, 1.0)
    s, t, w = brute.tuples_of(g)
    assert np.allclose(oracle.spmv(g, x), brute.spmv_dense(g.n, s, t, w, x), rtol=1e-13, atol=1e-13)


def test_spmv_ones_gives_weighted_degree():
    g = simgen.rmat(9, wmin=1, wmax=255)
    y = oracle.spmv(g, np.ones(g.n, np.float32))
    s, t, w = brute.tuples_of(g)
    wd = np.bincount(s, weights=w, minlength=g.n)  # symmetric: in-weight = out-weight
    assert np.array_equal(y, wd)
    gu = simgen.rmat(9)
    assert np.array_equal(oracle.spmv(gu, np.ones(gu.n, np.float32)), gu.degree().astype(np.float64))


# ---------------------------------------------------------------- BP (C-BP)
def test_bp_symmetric_prior_is_fixed_point():
    g = simgen.rmat(8, wmin=1, wmax=255)
    out = oracle.bp(g, np.full(g.n, 0.5, np.float32), 10)
    assert np.all(out == 0.0)


def test_bp_neutral_coupling_and_isolated():
    g = simgen.rmat(8, wmin=128, wmax=128)  # c = 0.25 + 0.5*127/254 = 0.5: psi uniform
    p = simgen.bp_prior(5, g.n)
    lp = np.log(p.astype(np.float64) / (1 - p.astype(np.float64)))
    assert np.allclose(oracle.bp(g, p, 10), lp, rtol=0, atol=1e-15)
    iso = simgen.from_edges(3, [(0, 1)])
    p3 = np.array([0.3, 0.6, 0.8], np.float32)
    out = oracle.bp(iso, p3, 5)
    assert abs(out[2] - math.log(0.8 / 0.2)) < 1e-7  # S:500 (p stored as f32)


def test_bp_two_vertex_closed_form():
    # unweighted edge (c = 0.75); p_a = 0.5, p_b = 0.9:
    # step 1: l(a) = 0 + log((.75*.9 + .25*.1)/(.75*.1 + .25*.9)) = log(0.7/0.3) = log(7/3)
    g = simgen.from_edges(2, [(0, 1)])
    p = np.array([0.5, 0.9], np.float32)
    out = oracle.bp(g, p, 1)
    pb = float(np.float32(0.9))
    exp_a = math.log((0.75 * pb + 0.25 * (1 - pb)) / (0.75 * (1 - pb) + 0.25 * pb))
    assert abs(out[0] - exp_a) < 1e-15
    assert abs(out[0] - math.log(7 / 3)) < 1e-6
    # b's neighbour a has b = 0.5 -> message log(1) = 0
    assert abs(out[1] - math.log(pb / (1 - pb))) < 1e-15


def test_bp_two_vertex_multi_step_closed_form():
    """T = 1, 2, 3 on one unweighted edge (c = 0.75), priors p_a = 0.75, p_b = 0.375
    (both exact in f32).  Derived by hand in the magnetisation form of the same
    recurrence (P:885 reading 15): with q = tanh(l/2) = 2b - 1 and theta = 2c - 1,
    log((c b + (1-c)(1-b)) / (c (1-b) + (1-c) b)) = 2 artanh(theta * q), so
    q_u' = (x_u + theta q_v) / (1 + x_u theta q_v), x_u = 2 p_u - 1 = tanh(logit(p_u)/2):
      x_a = 1/2, x_b = -1/4, theta = 1/2
      t=1: q_a = (1/2 - 1/8)/(1 - 1/16) = 2/5,   q_b = (-1/4 + 1/4)/(...) = 0
      t=2: q_a = 1/2,                            q_b = (-1/4 + 1/5)/(1 - 1/20) = -1/19
      t=3: q_a = (1/2 - 1/38)/(1 - 1/76) = 12/25, q_b = (-1/4 + 1/4)/(...) = 0
    and l = log((1+q)/(1-q)).  A recurrence that fed the prior (or the previous
    step's message alone) back instead of the current log-odds stops at t=1's
    values; one that swapped c and 1-c flips the signs."""
    g = simgen.from_edges(2, [(0, 1)])
    p = np.array([0.75, 0.375], np.float32)
    want = {1: (math.log(7 / 3), 0.0), 2: (math.log(3.0), math.log(9 / 10)), 3: (math.log(37 / 13), 0.0)}
    for T, (la, lb) in want.items():
        out = oracle.bp(g, p, T)
        assert abs(out[0] - la) < 1e-13 and abs(out[1] - lb) < 1e-13, (T, out, la, lb)


def test_bp_path3_multi_step_closed_form():
    """3-vertex path a - b - c with unequal couplings, T = 2 by hand (magnetisation
    form, see above).  Weights 255 (c = 3/4, theta = 1/2) on a-b and 1 (c = 1/4,
    theta = -1/2) on b-c; priors 0.75, 0.5, 0.25 -> x = (1/2, 0, -1/2).
      t=1: q_a = x_a + 0 = 1/2 (b's q is 0);  q_c = -1/2;
           q_b = tanh(0 + artanh(1/2 * 1/2) + artanh(-1/2 * -1/2)) = (1/4 + 1/4)/(1 + 1/16) = 8/17
      t=2: q_a = (1/2 + 1/2 * 8/17)/(1 + 1/2 * 1/2 * 8/17) = (25/34)/(19/17) = 25/38
           q_c = (-1/2 - 1/2 * 8/17)/(1 + (-1/2)(-1/2)(8/17)) = -25/38
           q_b = same as t=1 (a, c unchanged at t=1): 8/17
    l = log((1+q)/(1-q)): l_a(2) = log(63/13), l_c(2) = -log(63/13), l_b(2) = log(25/9)."""
    g = simgen.from_edges(3, [(0, 1), (1, 2)], [255, 1])
    p = np.array([0.75, 0.5, 0.25], np.float32)
    out = oracle.bp(g, p, 2)
    want = [math.log(63 / 13), math.log(25 / 9), -math.log(63 / 13)]
    assert np.allclose(out, want, rtol=0, atol=1e-13), (out, want)
    out1 = oracle.bp(g, p, 1)
    assert np.allclose(out1, [math.log(3.0), math.log(25 / 9), -math.log(3.0)], rtol=0, atol=1e-13)


def _bp_exact_rational(n, edges, weights, p, T):
    """Exact BP in rational arithmetic via the tanh rule (fractions.Fraction):
    q_u' = tanh(artanh(x_u) + sum_v artanh(theta_uv q_v)) folded with
    tanh(a + b) = (tanh a + tanh b) / (1 + tanh a tanh b); theta = 2c - 1 with
    c = 1/4 + (w-1)/508 (reading 15).  Independent of the oracle's log-ratio form."""
    from fractions import Fraction as F
    x = [F(float(pi)) * 2 - 1 for pi in p]
    nb = [[] for _ in range(n)]
    for (a, b), w in zip(edges, weights):
        th = 2 * (F(1, 4) + F(w - 1, 508)) - 1
        nb[a].append((b, th))
        nb[b].append((a, th))
    q = list(x)
    for _ in range(T):
        qn = []
        for u in range(n):
            s = x[u]
            for v, th in nb[u]:
                m = th * q[v]
                s = (s + m) / (1 + s * m)
            qn.append(s)
        q = qn
    return [math.log((1 + qi) / (1 - qi)) for qi in q]


def test_bp_loopy_graph_exact_rationals():
    """A triangle with a pendant and mixed couplings, T = 1..4, against exact
    rational BP (tanh rule): catches a wrong coupling map, a transposed message,
    or messages taken from the prior / previous message instead of the current
    log-odds at every step of a loopy recurrence."""
    edges = [(0, 1), (1, 2), (2, 0), (2, 3)]
    weights = [200, 40, 255, 1]
    p = np.array([0.625, 0.25, 0.875, 0.5], np.float32)
    g = simgen.from_edges(4, edges, weights)
    for T in (1, 2, 3, 4):
        want = _bp_exact_rational(4, edges, weights, p, T)
        assert np.allclose(oracle.bp(g, p, T), want, rtol=0, atol=1e-12), T


def test_bp_antisymmetry():
    # flipping every prior p -> 1-p negates every log-odds (psi is symmetric under x -> 1-x)
    g = simgen.rmat(8, wmin=1, wmax=255)
    p = simgen.bp_prior(9, g.n)
    a = oracle.bp(g, p, 6)
    b = oracle.bp(g, (1.0 - p.astype(np.float64)).astype(np.float32), 6)
    q = (1.0 - p.astype(np.float64)).astype(np.float32)
    # exact when 1-p is representable as computed; compare with a tolerance from the f32 round trip
    assert np.allclose(a, -b, rtol=1e-5, atol=1e-5)


# ---------------------------------------------------------------- WCC (C-W)
def test_wcc_closed_forms():
    """path -> one component labelled 0; isolated vertices keep their own id; two components -> 0 and 3."""
    g = simgen.from_edges(6, [(i, i + 1) for i in range(5)])
    assert list(oracle.wcc(g)) == [0] * 6
    g = simgen.from_edges(7, [(0, 1), (1, 2), (3, 4), (4, 5), (5, 6)])
    assert list(oracle.wcc(g)) == [0, 0, 0, 3, 3, 3, 3]
    g = simgen.from_edges(5, [(4, 2)])
    assert list(oracle.wcc(g)) == [0, 1, 2, 3, 2]
    assert list(oracle.wcc(simgen.from_edges(1, []))) == [0]


@pytest.mark.parametrize("seed", range(12))
def test_wcc_vs_scipy_components(seed):
    """The partition equals scipy's connected components; each label is the component's smallest id."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    n = 40 + 7 * seed
    g = simgen.random_graph(n, max(1, n // 2 + 3 * seed), seed)
    lab = oracle.wcc(g)
    A = csr_matrix((np.ones(g.m), g.col.astype(np.int64), g.row_ptr.astype(np.int64)), shape=(n, n))
    k, comp = connected_components(A, directed=False)
    for c in range(k):
        members = np.flatnonzero(comp == c)
        assert np.all(lab[members] == members.min())
    assert len(np.unique(lab)) == k


def test_wcc_invariants_rmat():
    """label(u) == label(v) on every edge, label(v) <= v, labels are fixed points."""
    g = simgen.rmat(12, 16, 3)
    lab = oracle.wcc(g)
    src = np.repeat(np.arange(g.n), np.diff(g.row_ptr.astype(np.int64)))
    assert np.all(lab[src] == lab[g.col])
    assert np.all(lab <= np.arange(g.n))
    assert np.all(lab[lab] == lab)
    # the component of vertex 0 is exactly the vertices BFS from 0 reaches
    reach = oracle.bfs(g, 0) != 0xFFFFFFFF
    assert np.array_equal(lab == 0, reach)
