"""k-core decomposition (R-MAT s24) with local chains of several lengths (device ms, median of 3)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import simgen  # noqa: E402
from paper_1812_04070_b200 import simdx  # noqa: E402

torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
d = simgen.rmat_gpu(24, 16, 1)
G = ctx.upload_device(d)
out = torch.empty(d.n, dtype=torch.int32, device="cuda:0")
ref = None
for lc in (0, 2, 8, 64, 100000):
    G.kcore(0, out=out, local_chain=lc)
    r = [G.kcore(0, out=out, local_chain=lc)[1] for _ in range(3)]
    o = out.cpu()
    ref = o if ref is None else ref
    print(f"local_chain={lc}: {statistics.median(x['ms'] for x in r):.2f} ms iters={r[0]['iterations']} same={bool((o == ref).all())}")
