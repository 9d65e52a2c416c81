import sys, numpy as np
sys.path.insert(0, '/root/repo')
import torch, oracle, simgen
from paper_1812_04070_b200 import simdx
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
for name, g in [("directed", simgen.random_graph(3000, 20000, 11, symmetric=False)), ("rmat12", simgen.rmat(12, 16, seed=2)),
                ("sym_rand", simgen.random_graph(3000, 20000, 11, symmetric=True))]:
    G = ctx.upload(g)
    for T in (1, 2, 5, 21):
        r, st, _ = G.pagerank_conv(0.85, 1e-300, T, 0, force_dir=2)
        o = oracle.pagerank(g, 0.85, T)
        rf, _, _ = G.pagerank(0.85, T)
        print(name, T, st["iterations"], "conv maxrel", np.max(np.abs(r - o) / o), "L1", np.abs(r - o).sum(), "sum", r.sum(),
              "| fixedT maxrel", np.max(np.abs(rf - o) / o))
    G.free()
