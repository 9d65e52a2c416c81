"""oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, single-threaded CPU reference for the SIMD-X ACC hot path
(arXiv 1812.04070; PAPER.md lines cited as P:<n>).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It shares no code with paper_1812_04070_b200 (the CUDA
path) and never imports it; its only inputs are simgen CSR graphs and vectors.

  bfs        C-B  queue BFS
  sssp       C-S  binary-heap Dijkstra
  coreness   C-K  Batagelj-Zaversnik buckets
  kcore_mask C-K  core(v) >= k
  pagerank   C-P  fp64 Jacobi, T steps          (reading 14)
  pagerank_conv C-PC fp64 Jacobi until L1 delta < eps (readings 25-26: both recurrences)
  spmv       C-V  fp64 y = A^T x over in-edges  (north_star)
  bp         C-BP fp64 log-odds Jacobi          (model = reading 15; T=1..4 closed forms)
  wcc        C-W  min vertex id per component   (P:345 names WCC)
  acc_model       the ACC BSP loop and its three filters on tiny graphs

All functions are pinned by tests/test_oracle.py (-m "not gpu").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None
INF = 0xFFFFFFFF


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        # -O2, no -ffast-math: fp64 arithmetic in program order
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", src, "-o", _SO, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        lib.oracle_bfs.argtypes = [u64, vp, vp, u32, vp]
        lib.oracle_sssp.argtypes = [u64, vp, vp, vp, i32, u32, vp]
        lib.oracle_coreness.argtypes = [u64, vp, vp, vp]
        lib.oracle_pagerank.argtypes = [u64, vp, vp, vp, ctypes.c_double, u32, vp]
        lib.oracle_pagerank_conv.argtypes = [u64, vp, vp, vp, ctypes.c_double, ctypes.c_double, u32, i32, vp,
                                             ctypes.POINTER(u32), ctypes.POINTER(ctypes.c_double)]
        lib.oracle_pagerank_conv.restype = ctypes.c_int
        lib.oracle_spmv.argtypes = [u64, vp, vp, vp, i32, vp, vp]
        lib.oracle_bp.argtypes = [u64, vp, vp, vp, i32, vp, u32, vp, vp]
        lib.oracle_wcc.argtypes = [u64, vp, vp, vp]
        for f in (lib.oracle_bfs, lib.oracle_sssp, lib.oracle_coreness, lib.oracle_pagerank,
                  lib.oracle_spmv, lib.oracle_bp):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _chk(rc, what):
    if rc == -1:
        raise ValueError(f"{what}: source out of range")
    if rc == -2:
        raise MemoryError(what)
    if rc == -3:
        raise ValueError(f"{what}: zero weight or distance overflow")


def _full(g):
    assert g.v_lo == 0 and g.v_hi == g.n, "oracle needs the whole graph"


def bfs(g, src: int) -> np.ndarray:
    _full(g)
    out = np.empty(g.n, np.uint32)
    _chk(_L().oracle_bfs(g.n, _p(g.row_ptr), _p(g.col), src, _p(out)), "bfs")
    return out


def sssp(g, src: int) -> np.ndarray:
    _full(g)
    out = np.empty(g.n, np.uint32)
    _chk(_L().oracle_sssp(g.n, _p(g.row_ptr), _p(g.col), _p(g.w), g.wbytes, src, _p(out)), "sssp")
    return out


def coreness(g) -> np.ndarray:
    _full(g)
    assert not g.directed, "k-core is defined on undirected graphs"
    out = np.empty(g.n, np.uint32)
    _chk(_L().oracle_coreness(g.n, _p(g.row_ptr), _p(g.col), _p(out)), "coreness")
    return out


def kcore_mask(g, k: int) -> np.ndarray:
    """1 if v is in the k-core (min degree >= k), else 0."""
    return (coreness(g) >= k).astype(np.uint32)


def pagerank(g, damping: float = 0.85, iters: int = 20) -> np.ndarray:
    _full(g)
    out = np.empty(g.n, np.float64)
    _chk(_L().oracle_pagerank(g.n, _p(g.row_ptr), _p(g.in_ptr()), _p(g.in_idx()), damping, iters, _p(out)),
         "pagerank")
    return out


def pagerank_conv(g, damping: float = 0.85, eps: float = 1e-6, max_iter: int = 1000, variant: int = 0):
    """oracle.c:oracle_pagerank_conv — Jacobi until the L1 change < eps.
    variant 0: normalised, dangling redistributed (reading 14); 1: SPEC S:487 (1-d) + d*sum, dangling dropped.
    Returns (ranks fp64, iterations, last L1 change)."""
    _full(g)
    out = np.empty(g.n, np.float64)
    it = ctypes.c_uint32()
    dl = ctypes.c_double()
    _chk(_L().oracle_pagerank_conv(g.n, _p(g.row_ptr), _p(g.in_ptr()), _p(g.in_idx()), damping, eps, max_iter,
                                   variant, _p(out), ctypes.byref(it), ctypes.byref(dl)), "pagerank_conv")
    return out, it.value, dl.value


def spmv(g, x: np.ndarray) -> np.ndarray:
    _full(g)
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty(g.n, np.float64)
    w = g.in_w()
    _chk(_L().oracle_spmv(g.n, _p(g.in_ptr()), _p(g.in_idx()), _p(w), 0 if w is None else w.dtype.itemsize,
                          _p(x), _p(out)), "spmv")
    return out


def bp(g, prior: np.ndarray, iters: int = 10, with_abs_terms: bool = False):
    _full(g)
    prior = np.ascontiguousarray(prior, np.float32)
    out = np.empty(g.n, np.float64)
    at = np.empty(g.n, np.float64)
    w = g.in_w()
    _chk(_L().oracle_bp(g.n, _p(g.in_ptr()), _p(g.in_idx()), _p(w), 0 if w is None else w.dtype.itemsize,
                        _p(prior), iters, _p(out), _p(at)), "bp")
    return (out, at) if with_abs_terms else out


def wcc(g) -> np.ndarray:
    """oracle.c:oracle_wcc — label(v) = smallest vertex id in v's connected component (undirected graphs)."""
    assert not getattr(g, "directed", False), "wcc: undirected graphs only"
    out = np.empty(g.n, np.uint32)
    _chk(_L().oracle_wcc(g.n, _p(g.row_ptr), _p(g.col), _p(out)), "wcc")
    return out


def level_histogram(level: np.ndarray) -> np.ndarray:
    """Per-level frontier sizes |F_0|, |F_1|, ... implied by BFS levels."""
    lv = level[level != INF].astype(np.int64)
    return np.bincount(lv) if lv.size else np.zeros(0, np.int64)


def traversed_edges(g, level: np.ndarray) -> int:
    """Graph500 m_cc: undirected edges in the traversed component = sum of reached degrees / 2."""
    deg = g.degree().astype(np.int64)
    return int(deg[level != INF].sum() // 2)
