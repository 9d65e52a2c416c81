"""Where the end-to-end step's time goes: upload of a pinned host CSR (H2D copy,
validation, degree arrays, workspace), the first BFS on the graph (includes the
one-off hub table), the level read-back and the free.
usage (GPU box): python profiles/e2e_probe.py [scale]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
d = simgen.rmat_gpu(scale, 16, 1)
host = d.to_host()
d.free()
n = host.n
rp = torch.from_numpy(host.row_ptr.view(np.int64)).pin_memory()
ci = torch.from_numpy(host.col.view(np.int32)).pin_memory()
out_h = torch.empty(n, dtype=torch.int32).pin_memory()
# raw H2D bandwidth for reference
dbuf = torch.empty(ci.numel(), dtype=torch.int32, device="cuda:0")
torch.cuda.synchronize()
t = time.perf_counter()
dbuf.copy_(ci, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"raw H2D copy of col: {ci.numel() * 4 / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
del dbuf
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = simdx.sx_graph_upload(ctx.h, n, rp, ci)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    G = simdx.Graph(ctx, h, n)
    G.bfs(0, out=out_h)
    t2 = time.perf_counter()
    G.bfs(0, out=out_h)
    t3 = time.perf_counter()
    G.free()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"rep {rep}: upload {1e3 * (t1 - t0):.1f} ms, first bfs (hub table + host levels) {1e3 * (t2 - t1):.1f} ms, "
          f"second bfs {1e3 * (t3 - t2):.1f} ms, free {1e3 * (t4 - t3):.1f} ms")
ctx.close()
