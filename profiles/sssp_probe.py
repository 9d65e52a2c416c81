"""SSSP on R-MAT: per-iteration timing across delta and direction modes.

usage (GPU box): python profiles/sssp_probe.py [scale] [deltas,...] [dirs,...] [cluster_enter,...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402
from probe import show  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
deltas = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 64, 256, 1024]
dirs = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
ces = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [2048]
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
d = simgen.rmat_gpu(scale, 16, 1, 1, 255)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
for ce in ces:
    for fd in dirs:
        for delta in deltas:
            G.sssp(0, delta, out=out, force_dir=fd, cluster_enter=ce)
            _, st, tr = G.sssp(0, delta, out=out, force_dir=fd, cluster_enter=ce, trace_cap=4096)
            show(f"sssp s{scale} delta={delta} force_dir={fd} cluster_enter={ce}", st, tr, 16)
G.free()
d.free()
ctx.close()
