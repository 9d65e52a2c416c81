"""The multi-GPU layer on one GPU: P virtual ranks run the
same partitioned kernels and exchange schedule with device copies in place of
the NCCL collectives.  Results must equal the oracle for every P."""
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


def build_dist(ctx, g, P):
    from paper_1812_04070_b200 import simdx
    D = simdx.Dist(ctx, g.n, P)
    for r in range(P):
        lo, hi = D.range(r)
        assert (lo, hi) == simdx.partition(g.n, P, r)
        rp = (g.row_ptr[lo:hi + 1] - g.row_ptr[lo]).astype(np.uint64)
        sl = simgen.CSR(n=g.n, row_ptr=rp, col=g.col[g.row_ptr[lo]:g.row_ptr[hi]].copy(),
                        w=None if g.w is None else g.w[g.row_ptr[lo]:g.row_ptr[hi]].copy(), v_lo=lo, v_hi=hi)
        D.upload(r, sl)
    return D


@pytest.fixture(scope="module")
def rmat14():
    return simgen.rmat(14, 16, seed=5, wmin=1, wmax=255)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_dist_bfs_rmat(ctx, rmat14, P):
    D = build_dist(ctx, rmat14, P)
    for src in (0, 1234):
        ref = oracle.bfs(rmat14, src)
        for mode in (dict(), dict(force_dir=1), dict(force_dir=2)):
            outs, st = D.bfs(src, **mode)
            assert np.array_equal(np.concatenate(outs), ref), (P, src, mode)
    D.free()


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_dist_sssp_rmat(ctx, rmat14, P):
    D = build_dist(ctx, rmat14, P)
    ref = oracle.sssp(rmat14, 0)
    for delta in (0, 64, 1024):
        outs, st = D.sssp(0, delta)
        assert np.array_equal(np.concatenate(outs), ref), (P, delta)
    D.free()


def test_dist_sssp_grid(ctx):
    g = simgen.grid(96, 80, seed=2)
    ref = oracle.sssp(g, 0)
    for P in (2, 5):
        D = build_dist(ctx, g, P)
        outs, _ = D.sssp(0, 512)
        assert np.array_equal(np.concatenate(outs), ref)
        outs, _ = D.bfs(0)
        assert np.array_equal(np.concatenate(outs), oracle.bfs(g, 0))
        D.free()


def test_dist_matches_single_gpu_at_scale20(ctx):
    g = simgen.rmat(20, 16, seed=1)
    ref = oracle.bfs(g, 0)
    D = build_dist(ctx, g, 4)
    outs, st = D.bfs(0)
    assert np.array_equal(np.concatenate(outs), ref)
    assert st["pull_iters"] >= 1  # the direction switch happens across ranks too
    D.free()


def test_dist_errors(ctx, rmat14):
    from paper_1812_04070_b200 import simdx
    with pytest.raises(simdx.SimdxError):
        simdx.Dist(ctx, rmat14.n, 4, 0, 2)  # nlocal must be 1 or nranks
    D = simdx.Dist(ctx, rmat14.n, 2)
    with pytest.raises(simdx.SimdxError):
        D.bfs(0)  # slices not uploaded
    D.free()


def test_dist_reupload_replaces_the_slices(ctx):
    """sx_dist_upload on an already loaded partition replaces the slices (bench.py's
    N-GPU e2e step re-uploads every step): BFS / SSSP answer for the new graph."""
    g1 = simgen.rmat(12, 16, seed=1, wmin=1, wmax=255)
    g2 = simgen.rmat(12, 8, seed=2, wmin=1, wmax=255)
    D = build_dist(ctx, g1, 4)
    outs, _ = D.bfs(0)
    assert np.array_equal(np.concatenate(outs), oracle.bfs(g1, 0))
    for rep in range(2):
        for r in range(4):
            lo, hi = D.range(r)
            rp = (g2.row_ptr[lo:hi + 1] - g2.row_ptr[lo]).astype(np.uint64)
            sl = simgen.CSR(n=g2.n, row_ptr=rp, col=g2.col[g2.row_ptr[lo]:g2.row_ptr[hi]].copy(),
                            w=g2.w[g2.row_ptr[lo]:g2.row_ptr[hi]].copy(), v_lo=lo, v_hi=hi)
            D.upload(r, sl)
        outs, _ = D.bfs(0)
        assert np.array_equal(np.concatenate(outs), oracle.bfs(g2, 0))
        outs, _ = D.sssp(0, 256)
        assert np.array_equal(np.concatenate(outs), oracle.sssp(g2, 0))
    D.free()


def test_dist_nccl_one_rank_communicator(ctx, rmat14):
    """The NCCL branch of the data path (allgather / alltoall / reduce-scatter /
    allreduce on a one-rank communicator) against the oracle."""
    from paper_1812_04070_b200 import simdx
    nid = simdx.sx_nccl_unique_id()
    D = simdx.Dist(ctx, rmat14.n, 1, 0, 1, nid)
    sl = simgen.CSR(n=rmat14.n, row_ptr=rmat14.row_ptr.copy(), col=rmat14.col.copy(), w=rmat14.w.copy(),
                    v_lo=0, v_hi=rmat14.n)
    D.upload(0, sl)
    for src in (0, 1234):
        ref = oracle.bfs(rmat14, src)
        for mode in (dict(), dict(force_dir=1), dict(force_dir=2)):
            outs, st = D.bfs(src, **mode)
            assert np.array_equal(outs[0], ref), (src, mode)
            # the device-initiated BFS (NCCL device API: symmetric window, LSA
            # stores and barrier inside one persistent kernel; §8(f) NEXT-1)
            outs, st = D.bfs(src, fusion=2, **mode)
            assert np.array_equal(outs[0], ref), ("fused", src, mode)
            assert st["launches"] == 1 and st["iterations"] == len(oracle.level_histogram(ref))
    # asynchronous device-initiated runs (sx_dist_bfs_async): enqueued back to back,
    # levels written in place into a device slice, statistics from sx_dist_sync
    import torch
    dev = torch.full((rmat14.n,), -7, dtype=torch.int32, device="cuda")
    for src in (1234, 0):
        D.bfs_async(src, [dev])
    st = D.sync()
    ref0 = oracle.bfs(rmat14, 0)
    assert np.array_equal(dev.cpu().numpy().view(np.uint32), ref0)
    assert st["runs"] == 2 and st["iterations"] == len(oracle.level_histogram(ref0)) and st["ms"] > 0
    with pytest.raises(simdx.SimdxError):
        D.bfs_async(0, [np.empty(rmat14.n, np.uint32)])  # host slice refused
    with pytest.raises(ValueError):
        D.bfs(0, outs=[np.empty(rmat14.n - 1, np.uint32)])  # short slice: checked before the C call
    with pytest.raises(ValueError):
        D.bfs(0, outs=[np.empty(rmat14.n, np.uint64)])  # 8-byte elements
    ref = oracle.sssp(rmat14, 0)
    for delta in (0, 1024):
        outs, _ = D.sssp(0, delta)
        assert np.array_equal(outs[0], ref), delta
    D.free()


@pytest.mark.parametrize("fusion", [1, 2])
def test_bench_dist_path_under_torchrun(fusion):
    """bench.py's multi-GPU path (torchrun, NCCL communicator, max-over-ranks
    timing) at one rank: one JSON line with the contract's keys.  fusion 2: the
    device-initiated BFS with asynchronous steps (sx_dist_bfs_async)."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "1", "--dist", "--scale", "16",
           "--steps", "3", "--warmup", "3", "--no-e2e", "--fusion", str(fusion)]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["unit"] == "GTEPS" and line["value"] > 0 and line["n_gpus"] == 1
    assert line["config"]["parallelism"] == "1d1" and "NCCL" in line["config"]["workload"]
    assert line["gpu_launches"] > 0
    if fusion == 2:
        assert "device API" in line["config"]["workload"] and line["gpu_launches"] == 3  # one kernel per step
