"""C2: iteration time vs frontier size (trace timestamps)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch, simgen
from paper_1812_04070_b200 import simdx
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
g = simgen.grid(2048, 2048, 1, 1, 255)
G = ctx.upload(g)
for delta in (1024, 4096):
    G.sssp(0, delta)
    _, st, tr = G.sssp(0, delta, trace_cap=20000)
    t = np.array([r["t_ns"] for r in tr], dtype=np.float64)
    dt = np.diff(t) / 1e3
    nf = np.array([r["n_frontier"] for r in tr][1:])
    act = np.array([sum(r["n_active"]) for r in tr][:-1])  # tasks processed in the next iteration
    filt = np.array([r["filter"] for r in tr][1:])
    print(f"delta={delta} iters={len(tr)} total={st['ms']:.1f} ms; mean dt={dt.mean():.1f} us")
    for lo, hi in ((0, 10), (10, 100), (100, 1000), (1000, 3000), (3000, 10000), (10000, 1 << 30)):
        m = (act >= lo) & (act < hi) & (filt == 0)
        if m.any():
            print(f"  tasks in [{lo},{hi}): n={m.sum():5d} dt mean={dt[m].mean():6.1f} us  p90={np.percentile(dt[m], 90):6.1f}")
    m = filt == 1
    print(f"  ballot/bucket iterations: n={m.sum()} dt mean={dt[m].mean() if m.any() else 0:.1f} us")
