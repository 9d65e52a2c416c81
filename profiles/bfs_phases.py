"""BFS s24 phase costs: time of a BFS cut after k iterations (max_iters=k), per k."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
d = simgen.rmat_gpu(int(sys.argv[1]) if len(sys.argv) > 1 else 24, 16, 1)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
for _ in range(3):
    G.bfs(0, out=out)
for k in range(1, 8):
    ms = []
    for _ in range(10):
        _, st, _ = G.bfs(0, out=out, max_iters=k)
        ms.append(st["ms"])
    print(f"max_iters={k}: device ms={np.median(ms):.4f} launches={st['launches']} push={st['ms_push']:.4f} pull={st['ms_pull']:.4f}")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(20):
        G.bfs(0, out=out)
    ev1.record()
    torch.cuda.synchronize()
    print(f"back-to-back full BFS: {ev0.elapsed_time(ev1) / 20:.4f} ms/call (device-measured stats ms {st['ms']:.4f})")
G.free()
ctx.close()
