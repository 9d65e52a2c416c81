"""Ablations of the paper's task-management and fusion choices on the synthetic
configs (the paper's Figs. 9, 12, 13):
JIT filter vs online-only vs ballot-only, selective fusion vs no fusion (one
launch per iteration), and the online-filter overflow threshold.  Device time
(CUDA events inside the call, graph resident), median of `reps` runs.
usage (GPU box): python profiles/ablation.py [reps]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)


def med(fn, **kw):
    fn(**kw)
    ts, st = [], None
    for _ in range(reps):
        _, st, _ = fn(**kw)
        ts.append(st["ms"])
    return statistics.median(ts), st


MODES = [("JIT (default)", {}), ("online only", dict(force_filter=1)), ("ballot only", dict(force_filter=2)),
         ("no fusion", dict(fusion=0)), ("JIT, no cluster tail", dict(cluster_enter=0))]


def table(name, fn, modes=MODES):
    print(f"\n== {name}")
    print(f"  {'mode':24s} {'ms':>10s} {'launches':>9s} {'iters':>7s} {'ballot':>7s}")
    base = None
    for label, kw in modes:
        ms, st = med(fn, **kw)
        base = base or ms
        print(f"  {label:24s} {ms:10.3f} {st['launches']:9d} {st['iterations']:7d} {st['ballot_iters']:7d}   x{ms / base:6.2f}")


g = simgen.rmat(16, 16, 1, 1, 255)
G = ctx.upload(g)
table("C1 BFS R-MAT s16 from 0", lambda **kw: G.bfs(0, **kw))
G.free()

d = simgen.rmat_gpu(24, 16, 1, 1, 255)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
table("BFS R-MAT s24 from 0 (bench workload)", lambda **kw: G.bfs(0, out=out, **kw))
print("\n== BFS s24: online-filter overflow threshold (P:649, Fig. 9)")
for thr in (8, 16, 32, 64, 128, 256):
    ms, st = med(lambda **kw: G.bfs(0, out=out, **kw), overflow_threshold=thr)
    print(f"  threshold {thr:4d}: {ms:8.3f} ms  ballot iters {st['ballot_iters']}")
table("SSSP R-MAT s24 from 0, delta 1024", lambda **kw: G.sssp(0, 1024, out=out, **kw), MODES[:4])
table("k-core decomposition R-MAT s24 (C4)", lambda **kw: G.kcore(0, out=out, **kw), MODES[:4])
G.free()

g = simgen.grid(2048, 2048, 1, 1, 255)
G = ctx.upload(g)
out = torch.empty(g.n, dtype=torch.int32, device="cuda:0")
table("C2 SSSP 2048^2 grid, delta 1024", lambda **kw: G.sssp(0, 1024, out=out, **kw))
print("\n== C2: online-filter overflow threshold")
for thr in (16, 64, 256):
    ms, st = med(lambda **kw: G.sssp(0, 1024, out=out, **kw), overflow_threshold=thr)
    print(f"  threshold {thr:4d}: {ms:8.3f} ms  ballot iters {st['ballot_iters']}")
G.free()
ctx.close()
