"""Host overhead of one sx_bfs call: wall time per call through the Python
binding, through a bare ctypes call with prebuilt arguments, and the device
time the call reports (usage: python profiles/host_probe.py [scale])."""
import ctypes
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
stream = torch.cuda.current_stream()
ctx = simdx.Context(0, stream.cuda_stream)
d = simgen.rmat_gpu(scale, 16, 1)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
for _ in range(5):
    G.bfs(0, out=out)
N = 200


def loop(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record(stream)
    for _ in range(N):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / N * 1e3, e0.elapsed_time(e1) / N


st = {}


def api():
    st["s"] = G.bfs(0, out=out)[1]


o = simdx.sx_opts()
simdx._lib.sx_opts_default(ctypes.byref(o))
s = simdx.sx_stats()
optr = ctypes.c_void_p(out.data_ptr())
fn = simdx._lib.sx_bfs
h = G.h


def bare():
    fn(h, 0, ctypes.byref(o), optr, ctypes.byref(s))


for name, f in (("api", api), ("bare", bare), ("api", api), ("bare", bare)):
    w, dv = loop(f)
    print(f"{name:5s}: wall {w:.4f} ms/call, events {dv:.4f} ms/call, device-reported {s.ms if name == 'bare' else st['s']['ms']:.4f} ms")
for mi in (1, 2):
    o.max_iters = mi
    w, dv = loop(bare)
    print(f"bare max_iters={mi}: wall {w:.4f} ms/call, events {dv:.4f} ms/call, device-reported {s.ms:.4f} ms")
for mode, name in ((0, "plain"), (1, "cooperative"), (2, "cluster16")):
    print(f"empty {name} launch: {simdx.sx_launch_bench(ctx.h, mode, 500):.2f} us")
