"""SSSP (delta 4096) and WCC on R-MAT (default s24) from vertex 0: device ms, best of 3, with the
library given by SIMDX_LIB; SX_MIN_HUBS=0 switches the frontier pulls' hub cache off.
usage: python profiles/sssp_time.py [scale]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
G = ctx.upload_device(simgen.rmat_gpu(scale, 16, 1, 1, 255))
out = torch.empty(1 << scale, dtype=torch.int32, device="cuda:0")
tag = f"{os.path.basename(os.environ.get('SIMDX_LIB', 'main'))} hubs={os.environ.get('SX_MIN_HUBS', '1')}"
G.sssp(0, 4096, out=out)
b = min((G.sssp(0, 4096, out=out)[1] for _ in range(3)), key=lambda s: s["ms"])
print(f"{tag}: sssp s{scale} delta=4096 {b['ms']:.2f} ms (push {b['ms_push']:.2f}, pull {b['ms_pull']:.2f}), {b['iterations']} it, {b['pull_iters']} pull")
G.wcc(out=out)
w = min((G.wcc(out=out)[1] for _ in range(3)), key=lambda s: s["ms"])
print(f"{tag}: wcc s{scale} {w['ms']:.2f} ms (push {w['ms_push']:.2f}, pull {w['ms_pull']:.2f}), {w['iterations']} it")
