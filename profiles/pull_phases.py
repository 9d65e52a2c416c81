"""Per-phase timing of the all-active pull (PageRank) from the device trace of a
-DSX_PULL_PHASES build: filter 7 = hub cache refreshed (CTA 0), 8 = phase A done,
1/2 = iteration done.  usage: SIMDX_LIB=build/libsimdx_phases.so python profiles/pull_phases.py [scale]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
G = ctx.upload_device(simgen.rmat_gpu(scale, 16, 1))
G.pagerank(0.85, 20)
_, st, tr = G.pagerank(0.85, 20, trace_cap=256)
print(f"pagerank s{scale}: ms={st['ms']:.3f}")
acc = {}
for a, b in zip(tr, tr[1:]):
    key = f"{a['filter']}->{b['filter']}"
    acc.setdefault(key, []).append((b["t_ns"] - a["t_ns"]) / 1e3)
for k, v in sorted(acc.items()):
    print(f"  {k:6s} n={len(v):3d} mean={sum(v) / len(v):9.1f} us  min={min(v):9.1f}")
