"""C2 (SSSP on the 2048^2 grid) time split from the device trace: iterations that
advanced the delta bucket (filter 1) vs plain iterations, by direction.
usage: python profiles/c2_phases.py [delta]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1812_04070_b200 import simdx  # noqa: E402

delta = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
G = ctx.grid(2048, 2048, 1, 1, 255)
out = torch.empty(2048 * 2048, dtype=torch.int32, device="cuda:0")
G.sssp(0, delta, out=out)
_, st, tr = G.sssp(0, delta, out=out, trace_cap=20000)
print(f"c2 delta={delta}: ms={st['ms']:.3f} iters={st['iterations']} records={len(tr)}")
acc = {}
for a, b in zip(tr, tr[1:]):
    key = (("push", "pull", "clus")[b["dir"]], b["filter"])
    acc.setdefault(key, []).append((b["t_ns"] - a["t_ns"]) / 1e3)
for k, v in sorted(acc.items()):
    v.sort()
    print(f"  {k}: n={len(v)} total={sum(v) / 1e3:.2f} ms mean={sum(v) / len(v):.2f} us median={v[len(v) // 2]:.2f} us")
