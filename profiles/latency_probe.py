"""Per-iteration fixed cost: SSSP / BFS / k-core on a path graph (frontier of one
vertex per iteration) vs the empty-barrier loop."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, simgen
from paper_1812_04070_b200 import simdx
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
us, ctas = simdx.sx_barrier_bench(ctx.h, 20000)
print(f"barrier: {us:.2f} us ({ctas} CTAs)")
L = 4000
g = simgen.from_edges(L, [(i, i + 1) for i in range(L - 1)], [1] * (L - 1))
G = ctx.upload(g)
for name, fn in (("bfs", lambda **k: G.bfs(0, **k)), ("sssp d=0", lambda **k: G.sssp(0, 0, **k)),
                 ("sssp d=2", lambda **k: G.sssp(0, 2, **k)), ("kcore", lambda **k: G.kcore(0, **k))):
    fn(force_dir=1)
    _, st, _ = fn(force_dir=1)
    print(f"{name:10s} path L={L}: {st['ms']:.2f} ms, {st['iterations']} iterations -> {1e3 * st['ms'] / max(1, st['iterations']):.2f} us/iteration, launches {st['launches']}")
G.free()
ctx.close()
