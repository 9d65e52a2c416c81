"""k-core decomposition on R-MAT s24 for several asynchronous thresholds
(cluster_enter) with the library given by SIMDX_LIB.  usage: python profiles/kcore_sweep.py [scale]"""
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
G = ctx.upload_device(simgen.rmat_gpu(scale, 16, 1))
out = torch.empty(1 << scale, dtype=torch.int32, device="cuda:0")
lib = os.path.basename(os.environ.get("SIMDX_LIB", "main"))
for ce in (0, 1024, 4096, 16384, 65536, 262144):
    G.kcore(0, out=out, cluster_enter=ce)
    ms = min(G.kcore(0, out=out, cluster_enter=ce)[1]["ms"] for _ in range(2))
    print(f"{lib}: kcore s{scale} cluster_enter={ce:7d}: {ms:.2f} ms")
