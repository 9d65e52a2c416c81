"""Host-side logic of the multi-GPU layer with a world-size-2 gloo group on CPU:
bootstrap (NCCL-id broadcast), the 1D partition rule, per-rank slice
generation, and the max/sum reductions bench.py uses."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    try:
        import simgen
        from paper_1812_04070_b200 import dist_host
        dist_host.init_group("gloo")
        # bootstrap: rank 0's id reaches every rank
        nid = dist_host.nccl_id_for_job(lambda: bytes(range(128)))
        # partition + slice generation
        scale = dist_host.weak_scale(8, world)
        n = 1 << scale
        lo, hi = dist_host.partition(n, world, rank)
        g = simgen.rmat(scale, 8, 11, 1, 255, v_lo=lo, v_hi=hi)
        t = dist_host.allreduce(float(rank + 1), "max")
        m = dist_host.allreduce(float(g.m), "sum")
        q.put((rank, nid, lo, hi, g.row_ptr.copy(), g.col.copy(), g.w.copy(), t, m, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, 0, 0, None, None, None, 0, 0, repr(e)))


@pytest.mark.parametrize("world", [2])
def test_gloo_bootstrap_partition_and_slices(world):
    import simgen
    from paper_1812_04070_b200 import dist_host
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[-1] is None, r[-1]
    # every rank got rank 0's id
    assert all(r[1] == bytes(range(128)) for r in res)
    # ranges tile [0, n) in rank order
    scale = dist_host.weak_scale(8, world)
    n = 1 << scale
    assert res[0][2] == 0 and res[-1][3] == n
    assert all(res[i][3] == res[i + 1][2] for i in range(world - 1))
    # the concatenated slices are the whole graph
    full = simgen.rmat(scale, 8, 11, 1, 255)
    col = np.concatenate([r[5] for r in res])
    w = np.concatenate([r[6] for r in res])
    deg = np.concatenate([np.diff(r[4]) for r in res])
    assert np.array_equal(col, full.col) and np.array_equal(w, full.w) and np.array_equal(deg, full.degree())
    # reductions
    assert all(r[7] == world for r in res)
    assert all(r[8] == full.m for r in res)


def test_partition_rule_matches_binding():
    from paper_1812_04070_b200 import dist_host, simdx
    for n, P in ((100, 3), (1 << 20, 8), (65, 2), (31, 4)):
        for r in range(P):
            assert dist_host.partition(n, P, r) == simdx.partition(n, P, r)
        lo0, _ = dist_host.partition(n, P, 0)
        assert lo0 == 0 and dist_host.partition(n, P, P - 1)[1] == n
        V = dist_host.partition(n, P, 0)[1]
        assert V % 32 == 0 or V == n
    assert dist_host.weak_scale(24, 8) == 27 and dist_host.weak_scale(24, 1) == 24
