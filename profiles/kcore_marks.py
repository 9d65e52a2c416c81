"""Anatomy of the asynchronous k-core levels (a -DSX_KCORE_MARKS build): from the
previous record to the end of the level start (5), then to CTA 0's view of the
cascade end (6), then to the level's closing barrier (4).
usage: SIMDX_LIB=build/libsimdx_kmarks.so python profiles/kcore_marks.py [scale]"""
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
G.kcore(0, out=out)
_, st, tr = G.kcore(0, out=out, trace_cap=20000)
a, b, c, seeds, items = [], [], [], [], []
for i in range(1, len(tr) - 2):
    if tr[i]["filter"] == 5 and tr[i + 1]["filter"] == 6 and tr[i + 2]["filter"] == 4:
        a.append((tr[i]["t_ns"] - tr[i - 1]["t_ns"]) / 1e3)
        b.append((tr[i + 1]["t_ns"] - tr[i]["t_ns"]) / 1e3)
        c.append((tr[i + 2]["t_ns"] - tr[i + 1]["t_ns"]) / 1e3)
        seeds.append(tr[i]["n_frontier"])
        items.append(tr[i + 1]["n_frontier"])
print(f"kcore s{scale}: ms {st['ms']:.2f}; speculative async levels {len(a)}")
for name, v in (("level start (scan + seed queue + barrier)", a), ("cascade (CTA 0 view)", b), ("to the closing barrier", c)):
    v = np.array(v)
    print(f"  {name:42s}: mean {v.mean():6.1f} us  median {np.median(v):6.1f}  p90 {np.percentile(v, 90):6.1f}")
print(f"  seeds per level: median {np.median(seeds):.0f}  mean {np.mean(seeds):.0f}; items CTA0 processed median {np.median(items):.0f}")
