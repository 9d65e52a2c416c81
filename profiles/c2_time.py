"""C2 SSSP on the 2048^2 grid: device time and iterations per delta (best of 3).
usage: [SIMDX_LIB=...] python profiles/c2_time.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1812_04070_b200 import simdx  # noqa: E402

torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
G = ctx.grid(2048, 2048, 1, 1, 255)
out = torch.empty(2048 * 2048, dtype=torch.int32, device="cuda:0")
for delta in (1024, 4096):
    G.sssp(0, delta, out=out)
    best = min((G.sssp(0, delta, out=out)[1] for _ in range(3)), key=lambda s: s["ms"])
    print(f"{os.path.basename(os.environ.get('SIMDX_LIB', 'main'))}: C2 delta={delta} {best['ms']:.2f} ms, "
          f"{best['iterations']} iterations, {best['ms'] * 1e3 / max(1, best['iterations']):.2f} us/iteration")
