"""GPU parity of the convergence runs (§8(f) NEXT-3): PageRank to convergence
with the pull -> push tail in both recurrences, and BP to convergence
(P:885), through the C ABI against the oracle.

PageRank: both recurrences are L1 contractions of factor d, so any iterate whose
unpropagated change is R lies within d/(1-d) * R of the fixed point; the oracle
at a 10^4 x tighter epsilon stands in for the fixed point.  The GPU result must
lie within d/(1-d) * (eps + eps_ref) of it (plus fp64 rounding) whatever mix of
pull steps and push-tail iterations ran; a pull-only run must reproduce the
oracle's own iteration count and values."""
import numpy as np
import pytest

import oracle
import simgen

pytestmark = pytest.mark.gpu
D = 0.85


@pytest.fixture(scope="module")
def ctx():
    import torch
    from paper_1812_04070_b200 import simdx
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    c = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
    yield c
    c.close()


def graphs():
    return {
        "rmat12": simgen.rmat(12, 16, seed=2),
        "rmat14": simgen.rmat(14, 16, seed=3),
        "directed": simgen.random_graph(3000, 20000, 11, symmetric=False),
        "star": simgen.from_edges(20001, [(0, i) for i in range(1, 20001)]),
        "path": simgen.from_edges(7, [(i, i + 1) for i in range(6)]),
        "single": simgen.from_edges(1, []),
    }


GS = graphs()


def scale_of(g, variant):
    return 1.0 if variant == 0 else float(g.n)  # L1 mass of the rank vector (variant 1: ~N)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("mode", [{}, dict(force_dir=1), dict(force_dir=2)], ids=["auto", "push_tail", "pull_only"])
@pytest.mark.parametrize("name", sorted(GS))
def test_pagerank_conv_bound(ctx, name, variant, mode):
    g = GS[name]
    eps = 1e-9 * scale_of(g, variant)
    G = ctx.upload(g)
    r, st, _ = G.pagerank_conv(D, eps, 100000, variant, **mode)
    ref, it_ref, _ = oracle.pagerank_conv(g, D, eps * 1e-4, 100000, variant)
    err = np.abs(r - ref).sum()
    bound = D / (1 - D) * (eps + eps * 1e-4) + 1e-12 * np.abs(ref).sum()
    assert err <= bound, (name, variant, mode, err, bound, st)
    assert st["residual"] <= eps, st
    if mode.get("force_dir") == 2:
        o, it_o, _ = oracle.pagerank_conv(g, D, eps, 100000, variant)
        assert st["iterations"] == it_o and st["launches"] == 1
        assert np.max(np.abs(r - o) / np.maximum(np.abs(o), 1e-300)) <= 1e-12
    if mode.get("force_dir") == 1 and g.n > 1:
        assert st["launches"] == 2 and st["pull_iters"] == 1  # one pull step, then the push tail
    if variant == 1:
        assert r.min() >= (1 - D) - 1e-12 * scale_of(g, variant)
    G.free()


def test_pagerank_conv_device_output_and_errors(ctx):
    import torch
    from paper_1812_04070_b200 import simdx
    g = GS["rmat12"]
    G = ctx.upload(g)
    out = torch.empty(g.n, dtype=torch.float64, device="cuda")
    _, st, _ = G.pagerank_conv(D, 1e-8, 100000, 0, out=out)
    ref, _, _ = oracle.pagerank_conv(g, D, 1e-12, 100000, 0)
    assert np.abs(out.cpu().numpy() - ref).sum() <= D / (1 - D) * 1.0001e-8 + 1e-12
    for bad in (dict(damping=1.0), dict(eps=0.0), dict(max_iters=0), dict(variant=2)):
        kw = dict(damping=D, eps=1e-8, max_iters=100, variant=0)
        kw.update(bad)
        with pytest.raises(simdx.SimdxError) as e:
            G.pagerank_conv(kw["damping"], kw["eps"], kw["max_iters"], kw["variant"])
        assert e.value.status == simdx.SX_E_INVALID
    with pytest.raises(ValueError):
        G.pagerank_conv(D, 1e-8, 100, 0, out=np.empty(g.n, np.float32))
    G.free()


def test_pagerank_conv_tail_runs_on_rmat(ctx):
    """R-MAT with both recurrences: auto mode (the decision tree picks pull or the
    tail) and the tail forced after one pull step both land within the bound."""
    g = simgen.rmat(16, 16, seed=1)
    G = ctx.upload(g)
    for var in (0, 1):
        eps = 1e-10 * scale_of(g, var)
        ref, _, _ = oracle.pagerank_conv(g, D, eps * 1e-4, 100000, var)
        for kw in ({}, dict(force_dir=1)):
            r, st, _ = G.pagerank_conv(D, eps, 100000, var, **kw)
            assert np.abs(r - ref).sum() <= D / (1 - D) * eps * 1.0001 + 1e-12 * ref.sum(), (var, kw, st)
            if kw:
                assert st["launches"] == 2 and st["pull_iters"] == 1 < st["iterations"], st
    G.free()


@pytest.mark.parametrize("name", ["rmat12", "directed", "path"])
def test_bp_conv(ctx, name):
    """BP to convergence = sx_bp's fixed-T recurrence with T = the first step whose
    L1 belief change is < eps (checked on the pinned fixed-T oracle)."""
    g = GS[name]
    if name == "directed":
        g = simgen.random_graph(3000, 20000, 11, wmin=1, wmax=255, symmetric=False)
    prior = simgen.bp_prior(5, g.n)
    eps = 1e-7 * g.n
    G = ctx.upload(g)
    lg, st, _ = G.bp_conv(prior, eps, 500)
    T = st["iterations"]
    assert 1 <= T < 500 and st["residual"] < eps
    o, terms = oracle.bp(g, prior, T, with_abs_terms=True)
    assert np.all(np.abs(lg - o) <= 1e-5 * (np.abs(o) + terms)), name

    def sig(x):
        return 1.0 / (1.0 + np.exp(-x))
    lp = np.log(prior.astype(np.float64) / (1 - prior.astype(np.float64)))
    prev = oracle.bp(g, prior, T - 1) if T > 1 else lp
    prev2 = oracle.bp(g, prior, T - 2) if T > 2 else lp
    d_last = np.abs(sig(o) - sig(prev)).sum()
    assert abs(d_last - st["residual"]) <= 1e-6 * max(eps, d_last)
    if T > 1:
        assert np.abs(sig(prev) - sig(prev2)).sum() >= eps * (1 - 1e-9)
    G.free()
