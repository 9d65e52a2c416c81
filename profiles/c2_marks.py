"""Anatomy of a C2 cluster-tail iteration (a -DSX_C2_MARKS build): SM cycles per segment of
thread 0's dependent chain, averaged over the iterations in which it had a task.
usage: SIMDX_LIB=build/libsimdx_c2marks.so python profiles/c2_marks.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1812_04070_b200 import simdx  # noqa: E402

torch.cuda.set_device(0)
ctx = simdx.Context(0, torch.cuda.current_stream().cuda_stream)
W = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
G = ctx.grid(W, W, 1, 1, 255)
out = torch.empty(W * W, dtype=torch.int32, device="cuda:0")
lib = simdx._lib
lib.sx_debug_c2_marks.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
G.sssp(0, 4096, out=out)
lib.sx_debug_c2_marks(buf, 1)
_, st, _ = G.sssp(0, 4096, out=out)
lib.sx_debug_c2_marks(buf, 1)
n = max(1, buf[9])
names = {1: "loop top -> list entry v", 2: "-> row bounds (rp)", 10: "-> ids", 11: "-> weights", 3: "-> dist(v)", 4: "-> atomicMin results",
         5: "-> append (returning atomic) + list store", 6: "-> flush far-min, arrive", 7: "cluster barrier",
         8: "-> counters after the barrier (vload)"}
print(f"grid {W}^2 delta=4096: {st['ms']:.2f} ms, {st['iterations']} iterations; thread 0 had a task in {buf[9]}")
tot = 0
for k in (1, 2, 10, 11, 3, 4, 5, 6, 7, 8):
    c = buf[k] / n
    tot += c
    print(f"  {names[k]:44s} {c:8.0f} cycles  {c / 1965:6.2f} us")
print(f"  {'sum':44s} {tot:8.0f} cycles  {tot / 1965:6.2f} us")
