"""Load balance of the BFS pull levels: per level, when each CTA finished its share
(globaltimer stamps of a -DSX_BFS_SPREAD build) relative to the first CTA.
usage: SIMDX_LIB=build/libsimdx_spread.so python profiles/bfs_spread.py [scale]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
G = ctx.upload_device(simgen.rmat_gpu(scale, 16, 1))
out = torch.empty(1 << scale, dtype=torch.int32, device="cuda:0")
cap = 32 + (8 * 4096 * 8) // 64 + 1  # trace records: 32 real + the stamp area (8 levels x 4096 CTAs x 8 B)
for _ in range(3):
    G.bfs(0, out=out, fusion=2, cluster_enter=0)
o = simdx.make_opts(fusion=2, cluster_enter=0)
buf = (simdx.sx_trace_rec * cap)()
o.trace = ctypes.cast(buf, ctypes.POINTER(simdx.sx_trace_rec))
o.trace_cap = cap
st = simdx.sx_bfs(G.h, 0, o, out, G.n)
raw = np.frombuffer(bytes(buf), dtype=np.uint64)[32 * 8:]  # records are 64 B = 8 x u64
grid = ctx.info()["sm_count"] * 3
for lv in range(8):
    t = raw[lv * 4096: lv * 4096 + grid]
    t = t[t > 0]
    if t.size < grid // 2:
        continue
    t = (t - t.min()) / 1e3
    print(f"pull level slot {lv}: CTAs {t.size}  finish spread: median {np.median(t):.1f} us  p90 {np.percentile(t, 90):.1f}  max {t.max():.1f}")
print("device ms", st.ms)
