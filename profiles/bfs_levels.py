"""Per-level device time of BFS from 0 on R-MAT (trace %globaltimer deltas, median of 20 runs)
for the library given by SIMDX_LIB (variant builds).
usage: SIMDX_LIB=build/libsimdx_<v>.so python profiles/bfs_levels.py [scale]"""
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
kw = {"fusion": int(os.environ["FUSION"])} if os.environ.get("FUSION") else {}
for _ in range(3):
    G.bfs(0, out=out, **kw)
runs = [G.bfs(0, out=out, trace_cap=64, **kw) for _ in range(20)]
ms = statistics.median(r[1]["ms"] for r in runs)
mp = statistics.median(r[1]["ms_pull"] for r in runs)
mpu = statistics.median(r[1]["ms_push"] for r in runs)
nl = min(len(r[2]) for r in runs)
dts = []
for i in range(1, nl):
    dts.append(statistics.median((r[2][i]["t_ns"] - r[2][i - 1]["t_ns"]) / 1e3 for r in runs))
tr = runs[0][2]
def _nm(t):
    return ('push', 'pull', 'clus')[t['dir']] if t['dir'] < 3 else f"mark{t['dir'] - 16}"
lv = " ".join(f"it{tr[i]['iter'] % 1000}:{_nm(tr[i])}:{dts[i - 1]:.1f}" for i in range(1, nl))
init = statistics.median(next((t["aux"] for t in r[2] if t["iter"] == 0 and t["dir"] == 0), 0) for r in runs) / 1e3
# (profiling builds: the iteration-0 record's aux = ns from the kernel start to the end of the state init)
if init > 0:
    lv = f"[init {init:.1f}] " + lv
print(f"{os.path.basename(os.environ.get('SIMDX_LIB', 'main'))} fusion={kw.get('fusion', 1)}: bfs s{scale} {ms * 1e3:.1f} us "
      f"(pull {mp * 1e3:.1f}, push {mpu * 1e3:.1f}) levels us: {lv}")
