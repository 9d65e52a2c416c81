import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, simgen
from paper_1812_04070_b200 import simdx
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
d = simgen.rmat_gpu(24, 16, 1)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
G.bfs(0, out=out, fusion=2)
_, st, tr = G.bfs(0, out=out, fusion=2, trace_cap=64)
for r in tr:
    print(r["iter"], r["dir"], r["filter"], list(r["n_active"]), r["n_frontier"], r["m_active"])
