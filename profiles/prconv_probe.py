"""PageRank to convergence on C3 (R-MAT s22): device time, pull steps, tail iterations
and residual for auto / pull-only / push-tail modes, both recurrences.
usage: python profiles/prconv_probe.py [scale]"""
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
n = 1 << scale
out = torch.empty(n, dtype=torch.float64, device="cuda:0")
for var, eps in ((0, 1e-6), (1, 1e-6 * n)):
    for name, kw in (("auto", {}), ("pull_only", dict(force_dir=2)), ("tail_after_1", dict(force_dir=1))):
        G.pagerank_conv(0.85, eps, 3000, var, out=out, **kw)
        _, st, _ = G.pagerank_conv(0.85, eps, 3000, var, out=out, **kw)
        print(f"variant {var} eps {eps:g} {name:12s}: {st['ms']:9.2f} ms  pull {st['pull_iters']:4d}  "
              f"total it {st['iterations']:5d}  launches {st['launches']}  residual {st['residual']:.3g}")
