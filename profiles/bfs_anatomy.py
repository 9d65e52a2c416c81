"""Anatomy of the first BFS pull level's TILE chunks (a -DSX_BFS_ANAT build): SM cycles per
segment, summed over CTA 0's warps, per chunk.  usage: SIMDX_LIB=build/libsimdx_anat.so
python profiles/bfs_anatomy.py [scale]"""
import ctypes
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
lib = simdx._lib
lib.sx_debug_bfs_anat.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
for _ in range(3):
    G.bfs(0, out=out, fusion=2)
lib.sx_debug_bfs_anat(buf, 1)
runs = 10
ms = 0.0
for _ in range(runs):
    ms += G.bfs(0, out=out, fusion=2)[1]["ms"]
lib.sx_debug_bfs_anat(buf, 1)
chunks = max(1, buf[7])
names = ["chunk claim -> visited / in-degree words", "scan + compaction into shared memory", "(unused)",
         "hub-first probe rounds", "row walks of the open candidates", "merge + stores of the chunk's words",
         "the next chunk's claim"]
print(f"bfs s{scale}: {ms / runs * 1e3:.1f} us per BFS; first pull level, CTA 0: {chunks / runs:.0f} chunks per BFS "
      f"over its 8 warps")
tot = 0
for k in (0, 1, 3, 4, 5, 6):
    c = buf[k] / chunks
    tot += c
    print(f"  {names[k]:44s} {c:8.0f} cycles per chunk  {c / 1965:6.2f} us")
print(f"  {'sum':44s} {tot:8.0f} cycles per chunk  {tot / 1965:6.2f} us")
