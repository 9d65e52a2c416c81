"""k-core decomposition trace (level starts, sub-rounds, asynchronous cascades) on
R-MAT, for two cluster_enter settings.  usage: python profiles/kcore_trace.py [scale] [nrec]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nrec = int(sys.argv[2]) if len(sys.argv) > 2 else 60
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
d = simgen.rmat_gpu(scale, 16, 1)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
res = {}
for ce in (0, 4096):
    G.kcore(0, out=out, cluster_enter=ce)
    _, st, tr = G.kcore(0, out=out, cluster_enter=ce, trace_cap=200000)
    res[ce] = out.cpu().numpy().copy()
    nls = sum(1 for t in tr if t["filter"] == 1)
    nas = sum(1 for t in tr if t["filter"] == 3)
    print(f"cluster_enter={ce}: ms={st['ms']:.2f} iters={st['iterations']} ballot={st['ballot_iters']} "
          f"records={len(tr)} level_starts~{nls} async={nas}")
    print("  " + " | ".join(f"{t['iter']}:f{t['filter']}:n{t['n_frontier']}:k{t['aux']}" for t in tr[:nrec]))
print("coreness equal:", np.array_equal(res[0], res[4096]))
