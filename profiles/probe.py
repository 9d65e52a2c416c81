"""Per-iteration timing probe (device %globaltimer in the trace) for the configs.

usage (on the GPU box): python profiles/probe.py [bfs24|c2|c3|c4|barrier|all]
Prints one line per iteration: direction, filter, |F'|, and the iteration's
duration from consecutive trace timestamps.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402


def show(name, st, tr, maxlines=40):
    print(f"== {name}: ms={st['ms']:.3f} launches={st['launches']} iters={st['iterations']} "
          f"ballot={st['ballot_iters']} pull={st['pull_iters']} edges={st['edges_examined']} "
          f"bytes={st['bytes_model'] / 1e6:.1f}MB ms_push={st['ms_push']:.3f} ms_pull={st['ms_pull']:.3f}")
    if not tr:
        return
    t0 = tr[0]["t_ns"]
    prev = None
    lines = []
    for t in tr:
        dt = (t["t_ns"] - prev) / 1e3 if prev is not None else float("nan")
        prev = t["t_ns"]
        lines.append(f"  it{t['iter']:5d} {('push', 'pull', 'clus')[t['dir']]} f{t['filter']} L{t['launch']} "
                     f"|F'|={t['n_frontier']:9d} act={t['n_active']} mf={t['m_active']} aux={t['aux']} dt={dt:8.1f}us")
    if len(lines) > maxlines:
        lines = lines[:maxlines // 2] + ["  ..."] + lines[-maxlines // 2:]
    print("\n".join(lines))
    print(f"  span first->last trace: {(tr[-1]['t_ns'] - t0) / 1e3:.1f} us over {len(tr)} records")


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    torch.cuda.set_device(0)
    ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
    if what in ("barrier", "all"):
        for it in (1000, 20000):
            us, ctas = simdx.sx_barrier_bench(ctx.h, it)
            print(f"== barrier: {us:.3f} us per grid barrier ({ctas} CTAs, {it} iterations)")
    if what in ("bfs24", "all"):
        g = simgen.rmat_gpu(24, 16, 1)
        G = ctx.upload_device(g)
        out = torch.empty(g.n, dtype=torch.int32, device="cuda:0")
        for _ in range(3):
            G.bfs(0, out=out)
        _, st, tr = G.bfs(0, out=out, trace_cap=64)
        show("bfs s24", st, tr)
        G.free()
    if what in ("c2", "all"):
        g = simgen.grid(2048, 2048, 1, 1, 255)
        G = ctx.upload(g)
        for delta in (0, 256, 1024, 4096):
            G.sssp(0, delta)
            _, st, tr = G.sssp(0, delta, trace_cap=8192)
            show(f"c2 sssp grid delta={delta}", st, tr, 12)
        G.free()
    if what in ("c3", "all"):
        g = simgen.rmat(22, 16, 1)
        G = ctx.upload(g)
        G.pagerank(0.85, 20)
        _, st, tr = G.pagerank(0.85, 20, trace_cap=64)
        show("c3 pagerank s22", st, tr, 8)
        G.free()
    if what in ("c4", "all"):
        g = simgen.rmat_gpu(24, 16, 1)
        G = ctx.upload_device(g)
        _, st, tr = G.kcore(0, trace_cap=8192)
        show("c4 kcore s24 k=0", st, tr, 16)
        _, st, tr = G.kcore(16, trace_cap=8192)
        show("c4 kcore s24 k=16", st, tr, 16)
        G.free()
    ctx.close()


if __name__ == "__main__":
    main()
