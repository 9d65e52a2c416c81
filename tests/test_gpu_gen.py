"""The GPU build of the input generator is bit-identical to simgen.c (so the
large bench graphs built on the GPU are the same graphs the oracle sees)."""
import numpy as np
import pytest

import simgen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale,wmax", [(10, 255), (13, 0), (14, 255), (12, 1000)])
def test_gpu_generator_matches_cpu(scale, wmax):
    wmin = 1 if wmax else 0
    cpu = simgen.rmat(scale, 16, 7, wmin, wmax)
    d = simgen.rmat_gpu(scale, 16, 7, wmin, wmax)
    gpu = d.to_host()
    d.free()
    assert np.array_equal(gpu.row_ptr, cpu.row_ptr)
    assert np.array_equal(gpu.col, cpu.col)
    if wmax:
        assert gpu.w.dtype == cpu.w.dtype and np.array_equal(gpu.w, cpu.w)
    else:
        assert gpu.w is None and cpu.w is None


def test_gpu_generator_slices():
    cpu = simgen.rmat(12, 16, 3, 1, 255)
    n = cpu.n
    for lo, hi in ((0, 1000), (1000, 2048), (2048, n)):
        d = simgen.rmat_gpu(12, 16, 3, 1, 255, v_lo=lo, v_hi=hi)
        s = d.to_host()
        d.free()
        assert np.array_equal(s.row_ptr, cpu.row_ptr[lo:hi + 1] - cpu.row_ptr[lo])
        assert np.array_equal(s.col, cpu.col[cpu.row_ptr[lo]:cpu.row_ptr[hi]])
        assert np.array_equal(s.w, cpu.w[cpu.row_ptr[lo]:cpu.row_ptr[hi]])


def test_upload_device_graph_and_dist_slices():
    import torch
    import oracle
    from paper_1812_04070_b200 import simdx
    torch.cuda.set_device(0)
    cpu = simgen.rmat(13, 16, 9, 1, 255)
    with simdx.Context(0, torch.cuda.current_stream().cuda_stream) as ctx:
        d = simgen.rmat_gpu(13, 16, 9, 1, 255)
        G = ctx.upload_device(d, borrow=True)
        lv, _, _ = G.bfs(0)
        assert np.array_equal(lv, oracle.bfs(cpu, 0))
        G.free()
        d.free()
        D = simdx.Dist(ctx, cpu.n, 4)
        slices = []
        for r in range(4):
            lo, hi = D.range(r)
            s = simgen.rmat_gpu(13, 16, 9, 1, 255, v_lo=lo, v_hi=hi)
            D.upload_device(r, s)
            slices.append(s)
        outs, _ = D.sssp(0, 1024)
        assert np.array_equal(np.concatenate(outs), oracle.sssp(cpu, 0))
        D.free()
        for s in slices:
            s.free()


def _ctx():
    import torch
    from paper_1812_04070_b200 import simdx
    torch.cuda.set_device(0)
    return simdx, simdx.Context(0, torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("scale,wmin,wmax,relabel", [(11, 1, 255, True), (12, 0, 0, True), (10, 1, 1000, True),
                                                     (9, 1, 255, False)])
def test_sx_graph_rmat_is_the_simgen_graph(scale, wmin, wmax, relabel):
    """sx_graph_rmat builds simgen.rmat's CSR on the device; sx_graph_download returns it."""
    simdx, ctx = _ctx()
    with ctx:
        cpu = simgen.rmat(scale, 16, 5, wmin, wmax, relabel_ids=relabel)
        G = ctx.rmat(scale, 16, 5, wmin, wmax, relabel=relabel)
        n, m, lo, hi = G.info()
        assert (n, m, lo, hi) == (cpu.n, cpu.m, 0, cpu.n)
        rp, col, w = G.download(weights=bool(wmax))
        assert np.array_equal(rp, cpu.row_ptr) and np.array_equal(col, cpu.col)
        if wmax:
            assert np.array_equal(w, cpu.w.astype(np.uint32))
        else:
            with pytest.raises(simdx.SimdxError) as e:
                G.download(weights=True)
            assert e.value.status == simdx.SX_E_WEIGHT
        G.free()


@pytest.mark.parametrize("rows,cols,wmax", [(1, 1, 255), (1, 9, 255), (7, 1, 255), (37, 53, 255), (64, 64, 0),
                                            (5, 6, 70000)])
def test_sx_graph_grid_is_the_simgen_grid(rows, cols, wmax):
    simdx, ctx = _ctx()
    with ctx:
        wmin = 1 if wmax else 0
        cpu = simgen.grid(rows, cols, 3, wmin, wmax)
        G = ctx.grid(rows, cols, 3, wmin, wmax)
        rp, col, w = G.download(weights=bool(wmax))
        assert np.array_equal(rp, cpu.row_ptr) and np.array_equal(col, cpu.col)
        if wmax:
            assert np.array_equal(w, cpu.w.astype(np.uint32))
        G.free()


def test_generated_graphs_run_the_path():
    """BFS on sx_graph_rmat and SSSP on sx_graph_grid agree with the oracle on the simgen graphs."""
    import oracle
    simdx, ctx = _ctx()
    with ctx:
        G = ctx.rmat(12, 16, 2, 1, 255)
        cpu = simgen.rmat(12, 16, 2, 1, 255)
        lv, _, _ = G.bfs(0)
        assert np.array_equal(lv, oracle.bfs(cpu, 0))
        G.free()
        G = ctx.grid(40, 70, 2, 1, 255)
        cpu = simgen.grid(40, 70, 2, 1, 255)
        d, _, _ = G.sssp(0, 256)
        assert np.array_equal(d, oracle.sssp(cpu, 0))
        G.free()


def test_generator_argument_errors():
    simdx, ctx = _ctx()
    with ctx:
        for args in ((0, 16, 1, 0, 0, 0), (10, 0, 1, 0, 0, 0), (10, 16, 1, 0, 5, 0), (10, 16, 1, 9, 5, 0),
                     (10, 16, 1, 0, 0, 8)):
            with pytest.raises(simdx.SimdxError) as e:
                simdx.sx_graph_rmat(ctx.h, *args)
            assert e.value.status == simdx.SX_E_INVALID
        with pytest.raises(simdx.SimdxError) as e:
            simdx.sx_graph_grid(ctx.h, 70000, 70000, 1, 1, 255)
        assert e.value.status == simdx.SX_E_INVALID
