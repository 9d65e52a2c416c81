"""simgen — seeded synthetic input generators (graphs + dense vectors).

The ONE module shared by the oracle side (tests/, oracle checks, bench's
cpu_baseline) and the CUDA side (bench, GPU tests): it holds none of the
method's arithmetic, only the inputs — CSR graphs shaped like the paper's
workloads (§6 Table 3; SURVEY.md §8(d) recipe) and input
vectors.  See simgen.c for the exact recipe.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsimgen.so")
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "simgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", src, "-o", _SO])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp = ctypes.c_void_p
        lib.simgen_philox.argtypes = [ctypes.c_uint32] * 4 + [ctypes.c_uint64, _u32p]
        lib.simgen_relabel.argtypes = [ctypes.c_uint64, ctypes.c_int]
        lib.simgen_relabel.restype = ctypes.c_uint64
        lib.simgen_rmat_tuples.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                           ctypes.c_uint32, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                           vp, vp, vp, vp]
        lib.simgen_csr_count.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, vp, vp,
                                         ctypes.c_int, vp]
        lib.simgen_csr_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, vp, vp, vp,
                                        ctypes.c_int, ctypes.c_int, vp, vp, vp]
        lib.simgen_csr_fill.restype = ctypes.c_int
        lib.simgen_grid_csr.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32,
                                        ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, vp, vp, vp,
                                        ctypes.c_int]
        lib.simgen_uniform_f32.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_float,
                                           ctypes.c_float, vp]
        _lib = lib
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


@dataclass
class CSR:
    """Host CSR graph: out-neighbour rows [v_lo, v_hi) of an n-vertex graph.

    row_ptr u64[nl+1] (local, starts at 0), col u32[m] (global ids), w u8/u32[m]
    or None.  For directed graphs csc_ptr/csc_idx/csc_w hold the in-neighbour
    rows; for undirected graphs they are None and the CSR
    serves as its own CSC.
    """
    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    w: Optional[np.ndarray] = None
    directed: bool = False
    csc_ptr: Optional[np.ndarray] = None
    csc_idx: Optional[np.ndarray] = None
    csc_w: Optional[np.ndarray] = None
    v_lo: int = 0
    v_hi: int = -1
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.v_hi < 0:
            self.v_hi = self.n

    @property
    def m(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def wbytes(self) -> int:
        return 0 if self.w is None else self.w.dtype.itemsize

    def degree(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def in_ptr(self):
        return self.row_ptr if self.csc_ptr is None else self.csc_ptr

    def in_idx(self):
        return self.col if self.csc_idx is None else self.csc_idx

    def in_w(self):
        return self.w if self.csc_idx is None else self.csc_w


# ---------------------------------------------------------------- GPU generator
_SO_GPU = os.path.join(_HERE, "libsimgen_gpu.so")
_lib_gpu = None


def build_gpu(force: bool = False) -> str:
    """nvcc-compile gpu_gen.cu (the same generator on the GPU) for sm_100a."""
    src = os.path.join(_HERE, "gpu_gen.cu")
    if force or not os.path.exists(_SO_GPU) or os.path.getmtime(_SO_GPU) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-std=c++17", "-Xcompiler", "-fPIC", "-shared", src, "-o", _SO_GPU])
    return _SO_GPU


def _LG():
    global _lib_gpu
    if _lib_gpu is None:
        build_gpu()
        lib = ctypes.CDLL(_SO_GPU)
        vp = ctypes.c_void_p
        lib.simgen_gpu_rmat_csr.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                            ctypes.c_uint32, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, vp,
                                            ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                            ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_int)]
        lib.simgen_gpu_rmat_csr.restype = ctypes.c_int
        lib.simgen_gpu_free.argtypes = [vp]
        lib.simgen_gpu_free.restype = None
        lib.simgen_gpu_to_host.argtypes = [vp, vp, ctypes.c_uint64]
        lib.simgen_gpu_to_host.restype = ctypes.c_int
        _lib_gpu = lib
    return _lib_gpu


class DeviceCSR:
    """Rows [v_lo, v_hi) of a graph in device memory (raw cudaMalloc pointers)."""

    def __init__(self, n, v_lo, v_hi, row_ptr, col, w, m, wbytes):
        self.n, self.v_lo, self.v_hi = n, v_lo, v_hi
        self.row_ptr_ptr, self.col_ptr, self.w_ptr = row_ptr, col, w
        self.m, self.wbytes = m, wbytes

    def to_host(self) -> CSR:
        L = _LG()
        nl = self.v_hi - self.v_lo
        rp = np.empty(nl + 1, np.uint64)
        col = np.empty(self.m, np.uint32)
        L.simgen_gpu_to_host(_p(rp), self.row_ptr_ptr, rp.nbytes)
        if self.m:
            L.simgen_gpu_to_host(_p(col), self.col_ptr, col.nbytes)
        w = None
        if self.wbytes:
            w = np.empty(self.m, np.uint8 if self.wbytes == 1 else np.uint32)
            if self.m:
                L.simgen_gpu_to_host(_p(w), self.w_ptr, w.nbytes)
        return CSR(n=self.n, row_ptr=rp, col=col, w=w, v_lo=self.v_lo, v_hi=self.v_hi)

    def free(self):
        L = _LG()
        for p in (self.row_ptr_ptr, self.col_ptr, self.w_ptr):
            if p:
                L.simgen_gpu_free(p)
        self.row_ptr_ptr = self.col_ptr = self.w_ptr = None


def rmat_gpu(scale: int, ef: int = 16, seed: int = 1, wmin: int = 0, wmax: int = 0, relabel_ids: bool = True,
             v_lo: int = 0, v_hi: Optional[int] = None, stream: int = 0) -> DeviceCSR:
    """rmat(...) built on the current CUDA device (bit-identical CSR, tests/test_gpu_gen.py)."""
    n = 1 << scale
    v_hi = n if v_hi is None else v_hi
    rp, col, w = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    m, wb = ctypes.c_uint64(), ctypes.c_int()
    rc = _LG().simgen_gpu_rmat_csr(scale, ef, seed, wmin, wmax, int(relabel_ids), v_lo, v_hi,
                                   ctypes.c_void_p(stream) if stream else None, ctypes.byref(rp), ctypes.byref(col),
                                   ctypes.byref(w), ctypes.byref(m), ctypes.byref(wb))
    if rc != 0:
        raise RuntimeError("simgen_gpu_rmat_csr failed (see stderr)")
    return DeviceCSR(n, v_lo, v_hi, rp.value, col.value, w.value, m.value, wb.value)


def philox(c0: int, c1: int, c2: int, c3: int, seed: int) -> tuple:
    out = (ctypes.c_uint32 * 4)()
    _L().simgen_philox(c0, c1, c2, c3, seed, out)
    return tuple(out)


def relabel(x: int, bits: int) -> int:
    return int(_L().simgen_relabel(x, bits))


def _wdtype(wmin: int, wmax: int):
    if wmax == 0 and wmin == 0:
        return None
    return np.uint8 if wmax <= 255 else np.uint32


def rmat_tuples(scale: int, ef: int = 16, seed: int = 1, wmin: int = 0, wmax: int = 0,
                relabel_ids: bool = True, lo: int = 0, hi: Optional[int] = None):
    m = ef << scale
    hi = m if hi is None else hi
    k = hi - lo
    src = np.empty(k, np.uint32)
    dst = np.empty(k, np.uint32)
    wdt = _wdtype(wmin, wmax)
    w = None if wdt is None else np.empty(k, wdt)
    _L().simgen_rmat_tuples(scale, ef, seed, wmin, wmax, int(relabel_ids), lo, hi, _p(src), _p(dst),
                            _p(w) if wdt is np.uint8 else None, _p(w) if wdt is np.uint32 else None)
    return src, dst, w


def csr_from_tuples(n: int, src: np.ndarray, dst: np.ndarray, w: Optional[np.ndarray] = None,
                    symmetric: bool = True, v_lo: int = 0, v_hi: Optional[int] = None) -> CSR:
    """Symmetrise (if requested), drop self-loops, keep duplicates, sort rows by (col, w)."""
    v_hi = n if v_hi is None else v_hi
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    if w is not None:
        w = np.ascontiguousarray(w)
        assert w.dtype in (np.uint8, np.uint32)
    m = src.shape[0]
    rp = np.empty(v_hi - v_lo + 1, np.uint64)
    _L().simgen_csr_count(v_lo, v_hi, m, _p(src), _p(dst), int(symmetric), _p(rp))
    nnz = int(rp[-1])
    col = np.empty(nnz, np.uint32)
    wo = None if w is None else np.empty(nnz, w.dtype)
    rc = _L().simgen_csr_fill(v_lo, v_hi, m, _p(src), _p(dst), _p(w), 0 if w is None else w.dtype.itemsize,
                              int(symmetric), _p(rp), _p(col), _p(wo))
    if rc != 0:
        raise MemoryError("simgen_csr_fill: out of host memory")
    g = CSR(n=n, row_ptr=rp, col=col, w=wo, directed=not symmetric, v_lo=v_lo, v_hi=v_hi)
    if not symmetric and v_lo == 0 and v_hi == n:
        # in-neighbour rows (CSC) for pull on directed graphs
        cp = np.empty(n + 1, np.uint64)
        _L().simgen_csr_count(0, n, m, _p(dst), _p(src), 0, _p(cp))
        ci = np.empty(int(cp[-1]), np.uint32)
        cw = None if w is None else np.empty(int(cp[-1]), w.dtype)
        _L().simgen_csr_fill(0, n, m, _p(dst), _p(src), _p(w), 0 if w is None else w.dtype.itemsize, 0,
                             _p(cp), _p(ci), _p(cw))
        g.csc_ptr, g.csc_idx, g.csc_w = cp, ci, cw
    return g


def rmat(scale: int, ef: int = 16, seed: int = 1, wmin: int = 0, wmax: int = 0,
         relabel_ids: bool = True, v_lo: int = 0, v_hi: Optional[int] = None) -> CSR:
    """Undirected Graph500-style R-MAT graph with 2^scale vertices, ef*2^scale tuples."""
    n = 1 << scale
    src, dst, w = rmat_tuples(scale, ef, seed, wmin, wmax, relabel_ids)
    g = csr_from_tuples(n, src, dst, w, True, v_lo, v_hi)
    g.meta = dict(kind="rmat", scale=scale, ef=ef, seed=seed, wmin=wmin, wmax=wmax)
    return g


def grid(rows: int, cols: int, seed: int = 1, wmin: int = 1, wmax: int = 255,
         v_lo: int = 0, v_hi: Optional[int] = None) -> CSR:
    """rows x cols 4-neighbour grid ("road-like", high diameter)."""
    n = rows * cols
    v_hi = n if v_hi is None else v_hi
    nl = v_hi - v_lo
    rp = np.empty(nl + 1, np.uint64)
    # closed-form degree upper bound for allocation: 4 per vertex
    col = np.empty(4 * nl, np.uint32)
    wdt = _wdtype(wmin, wmax)
    w = None if wdt is None else np.empty(4 * nl, wdt)
    _L().simgen_grid_csr(rows, cols, seed, wmin, wmax, v_lo, v_hi, _p(rp), _p(col), _p(w),
                         0 if w is None else w.dtype.itemsize)
    nnz = int(rp[-1])
    g = CSR(n=n, row_ptr=rp, col=col[:nnz].copy(), w=None if w is None else w[:nnz].copy(),
            v_lo=v_lo, v_hi=v_hi)
    g.meta = dict(kind="grid", rows=rows, cols=cols, seed=seed, wmin=wmin, wmax=wmax)
    return g


def from_edges(n: int, edges, weights=None, symmetric: bool = True) -> CSR:
    """Tiny explicit graphs (tests, Fig. 1 fixture)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    w = None
    if weights is not None:
        wv = np.asarray(weights, dtype=np.int64)
        w = wv.astype(np.uint8) if (wv.size == 0 or wv.max() <= 255) else wv.astype(np.uint32)
    return csr_from_tuples(n, e[:, 0].astype(np.uint32), e[:, 1].astype(np.uint32), w, symmetric)


def random_graph(n: int, m: int, seed: int, wmin: int = 0, wmax: int = 0, symmetric: bool = True) -> CSR:
    """Uniform random multigraph with m tuples (tiny brute-force cases)."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m, dtype=np.int64) if n > 0 else np.zeros(0, np.int64)
    dst = rng.integers(0, n, m, dtype=np.int64) if n > 0 else np.zeros(0, np.int64)
    w = None
    if wmax:
        w = rng.integers(wmin, wmax + 1, m, dtype=np.int64)
        w = w.astype(np.uint8 if wmax <= 255 else np.uint32)
    return csr_from_tuples(n, src.astype(np.uint32), dst.astype(np.uint32), w, symmetric)


def uniform_f32(seed: int, stream: int, n: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(n, np.float32)
    _L().simgen_uniform_f32(seed, stream, n, lo, hi, _p(out))
    return out


def bp_prior(seed: int, n: int) -> np.ndarray:
    """BP priors p_u ~ U[0.1, 0.9] (SURVEY.md §8(c) C-BP reading)."""
    return uniform_f32(seed, 0xB9, n, 0.1, 0.9)
