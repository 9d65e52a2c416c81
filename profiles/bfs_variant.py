"""Device time of BFS from 0 on R-MAT s24 for the library given by SIMDX_LIB (variant builds).
usage: SIMDX_LIB=build/libsimdx_<v>.so python profiles/bfs_variant.py [scale]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
d = simgen.rmat_gpu(scale, 16, 1)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
for _ in range(5):
    G.bfs(0, out=out)
st = [G.bfs(0, out=out)[1] for _ in range(30)]
ms = statistics.median(s["ms"] for s in st)
mp = statistics.median(s["ms_pull"] for s in st)
mpu = statistics.median(s["ms_push"] for s in st)
print(f"{os.path.basename(os.environ.get('SIMDX_LIB', 'main'))}: bfs s{scale} {ms * 1e3:.1f} us (pull {mp * 1e3:.1f}, push {mpu * 1e3:.1f})")
