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
