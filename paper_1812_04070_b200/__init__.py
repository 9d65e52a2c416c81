"""paper_1812_04070_b200 — B200-native SIMD-X ACC frontier engine (arXiv 1812.04070).

The hot path (ACC frontier step: JIT online/ballot filters, thread/warp/CTA
binning, push/pull switch, fused persistent kernels with a grid barrier) lives
in libsimdx.so (csrc/, sm_100a CUDA) behind the C ABI in include/simdx.h;
`simdx` is its ctypes binding.  Importing this package fails loudly if the
extension has not been built — there is no CPU fallback.
"""
from . import simdx  # noqa: F401
from .simdx import Context, Graph, SimdxError  # noqa: F401

__all__ = ["simdx", "Context", "Graph", "SimdxError"]
