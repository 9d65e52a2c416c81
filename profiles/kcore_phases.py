"""k-core decomposition time split from the device trace: level starts (min
scan + ballot filter of the seeds: records with filter 1) vs cascade sub-rounds
(filter 0), with frontier-size buckets.  usage: python profiles/kcore_phases.py [scale]"""
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
d = simgen.rmat_gpu(scale, 16, 1)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
G.kcore(0, out=out)
_, st, tr = G.kcore(0, out=out, trace_cap=8192)
print(f"kcore s{scale}: ms={st['ms']:.3f} records={len(tr)} iters={st['iterations']} ballot={st['ballot_iters']}")
lvl, sub, alv, acas = [], {}, [], []
for a, b in zip(tr, tr[1:]):
    dt = (b["t_ns"] - a["t_ns"]) / 1e3
    if b["filter"] == 1:
        lvl.append(dt)  # previous record -> level start done
    elif b["filter"] == 4:
        alv.append(dt)  # a whole level run asynchronously (level start + queue)
    elif b["filter"] == 3:
        acas.append(dt)  # the asynchronous rest of a level's cascade
    else:
        nf = a["n_frontier"]
        key = "<=1e2" if nf <= 100 else "<=1e4" if nf <= 10000 else "<=1e6" if nf <= 1000000 else ">1e6"
        sub.setdefault(key, []).append(dt)
print(f"  level starts: n={len(lvl)} total={sum(lvl) / 1e3:.2f} ms mean={sum(lvl) / max(1, len(lvl)):.1f} us")
for name, v in (("asynchronous levels", alv), ("asynchronous cascade tails", acas)):
    if v:
        print(f"  {name}: n={len(v)} total={sum(v) / 1e3:.2f} ms mean={sum(v) / len(v):.1f} us")
for k, v in sorted(sub.items()):
    print(f"  sub-rounds with |F| {k}: n={len(v)} total={sum(v) / 1e3:.2f} ms mean={sum(v) / len(v):.1f} us")
