"""Cost of the small-frontier cluster mode's pieces (sx_cluster_bench) on one 16-CTA cluster."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1812_04070_b200 import simdx  # noqa: E402

torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
print(f"empty cluster launch: {simdx.sx_cluster_bench(ctx.h, 256, 0, 200):.2f} us")
print(f"cluster barrier:      {simdx.sx_cluster_bench(ctx.h, 256, 1, 20000):.3f} us")
for nw in (1 << 12, 1 << 15, 1 << 17, 1 << 19):
    z = simdx.sx_cluster_bench(ctx.h, nw, 2, 100)
    zc = simdx.sx_cluster_bench(ctx.h, nw, 3, 100)
    print(f"nwords={nw:8d} ({nw * 4 / 1e6:.2f} MB): zero {z:7.2f} us   zero+compact {zc:7.2f} us")
ctx.close()
