"""C3 PageRank (R-MAT s22, 20 iterations) device time for the library given by
SIMDX_LIB (variant builds), best of 3.  usage: SIMDX_LIB=... python profiles/pr_variants.py [scale]"""
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
out = torch.empty(1 << scale, dtype=torch.float32, device="cuda:0")
G.pagerank(0.85, 20, out=out)
ms = min(G.pagerank(0.85, 20, out=out)[1]["ms"] for _ in range(3))
print(f"{os.path.basename(os.environ.get('SIMDX_LIB', 'main'))}: pagerank s{scale} x20 {ms:.3f} ms")
