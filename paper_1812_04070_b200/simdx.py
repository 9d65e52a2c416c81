"""ctypes binding of include/simdx.h — argument marshalling only.

Every step of the hot path runs in libsimdx.so (hand-written sm_100a CUDA);
this module only converts numpy arrays / torch tensors to pointers and status
codes to exceptions.  There is NO fallback: if the extension is missing this
module raises at import time, and on a machine without a B200 every call
returns SX_E_CUDA.

Function names follow the C ABI (sx_ctx_create, sx_graph_upload, sx_bfs, ...);
`Context` / `Graph` are thin conveniences over them.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SIMDX_LIB") or os.path.join(_HERE, "libsimdx.so")  # SIMDX_LIB: variant builds (profiles/)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build the CUDA extension first "
                      "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants
SX_OK, SX_E_INVALID, SX_E_OOM, SX_E_CUDA, SX_E_NCCL, SX_E_NO_REVERSE, SX_E_WEIGHT, SX_E_BARRIER, SX_E_STATE = range(9)
SX_DIRECTED, SX_DEVICE_PTRS, SX_BORROW, SX_DEDUP = 1, 2, 4, 8
INF = 0xFFFFFFFF

_u64, _u32, _i32, _f32, _vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_float, ctypes.c_void_p


class sx_csr_desc(ctypes.Structure):
    _fields_ = [("n", _u64), ("m", _u64), ("row_ptr", _vp), ("col", _vp), ("w", _vp), ("w_bytes", _u32),
                ("csc_ptr", _vp), ("csc_idx", _vp), ("csc_w", _vp), ("flags", _u32)]


class sx_trace_rec(ctypes.Structure):
    _fields_ = [("iter", _u32), ("dir", _u32), ("filter", _u32), ("launch", _u32), ("n_active", _u32 * 4),
                ("n_frontier", _u64), ("m_active", _u64), ("aux", _u64), ("t_ns", _u64)]


class sx_opts(ctypes.Structure):
    _fields_ = [("overflow_threshold", _u32), ("sep_small", _u32), ("sep_large", _u32), ("sep_huge", _u32),
                ("alpha", _f32), ("beta", _f32), ("force_filter", _i32), ("force_dir", _i32), ("fusion", _i32),
                ("max_iters", _u32), ("trace", ctypes.POINTER(sx_trace_rec)), ("trace_cap", _u64),
                ("local_chain", _u32), ("cluster_enter", _u32)]


class sx_stats(ctypes.Structure):
    _fields_ = [("iterations", _u32), ("launches", _u32), ("ballot_iters", _u32), ("pull_iters", _u32),
                ("edges_examined", _u64), ("vertices_scanned", _u64), ("list_entries", _u64),
                ("bytes_model", ctypes.c_double), ("ms", ctypes.c_double), ("ms_push", ctypes.c_double),
                ("ms_pull", ctypes.c_double), ("bytes_push", ctypes.c_double), ("bytes_pull", ctypes.c_double),
                ("launches_push", _u32), ("launches_pull", _u32), ("ms_fused", ctypes.c_double),
                ("launches_fused", _u32), ("runs", _u32), ("residual", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class sx_device_info(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int) for k in ("device", "sm_count", "cc_major", "cc_minor", "regs_per_sm",
                                            "max_threads_per_sm", "block_threads", "push_ctas_per_sm",
                                            "pull_ctas_per_sm", "push_regs", "pull_regs")]


_P = ctypes.POINTER
_lib.sx_status_str.argtypes = [ctypes.c_int]
_lib.sx_status_str.restype = ctypes.c_char_p
_lib.sx_last_error.argtypes = []
_lib.sx_last_error.restype = ctypes.c_char_p
_lib.sx_version.restype = ctypes.c_int
_lib.sx_ctx_create.argtypes = [ctypes.c_int, _vp, _P(_vp)]
_lib.sx_ctx_destroy.argtypes = [_vp]
_lib.sx_ctx_destroy.restype = None
_lib.sx_ctx_info.argtypes = [_vp, _P(sx_device_info)]
_lib.sx_graph_upload.argtypes = [_vp, _P(sx_csr_desc), _P(_vp)]
_lib.sx_graph_info.argtypes = [_vp, _P(_u64), _P(_u64), _P(_u64), _P(_u64)]
_lib.sx_graph_free.argtypes = [_vp]
_lib.sx_graph_rmat.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _u64, _u32, _u32, _u32, _P(_vp)]
_lib.sx_graph_grid.argtypes = [_vp, _u32, _u32, _u64, _u32, _u32, _P(_vp)]
_lib.sx_graph_download.argtypes = [_vp, _vp, _vp, _vp]
_lib.sx_graph_free.restype = None
_lib.sx_opts_default.argtypes = [_P(sx_opts)]
_lib.sx_opts_default.restype = None
_lib.sx_bfs.argtypes = [_vp, _u32, _P(sx_opts), _vp, _P(sx_stats)]
_lib.sx_bfs_async.argtypes = [_vp, _u32, _P(sx_opts), _vp]
_lib.sx_graph_sync.argtypes = [_vp, _P(sx_stats)]
_lib.sx_barrier_fault.argtypes = [_vp, _u32, _u32]
_lib.sx_sssp.argtypes = [_vp, _u32, _u32, _P(sx_opts), _vp, _P(sx_stats)]
_lib.sx_pagerank.argtypes = [_vp, _f32, _u32, _P(sx_opts), _vp, _P(sx_stats)]
_lib.sx_pagerank_conv.argtypes = [_vp, ctypes.c_double, ctypes.c_double, _u32, _u32, _P(sx_opts), _vp, _P(sx_stats)]
_lib.sx_bp_conv.argtypes = [_vp, _vp, ctypes.c_double, _u32, _P(sx_opts), _vp, _P(sx_stats)]
_lib.sx_kcore.argtypes = [_vp, _u32, _P(sx_opts), _vp, _P(sx_stats)]
_lib.sx_spmv.argtypes = [_vp, _vp, _u32, _P(sx_opts), _vp, _P(sx_stats)]
_lib.sx_bp.argtypes = [_vp, _vp, _u32, _P(sx_opts), _vp, _P(sx_stats)]
_lib.sx_wcc.argtypes = [_vp, _P(sx_opts), _vp, _P(sx_stats)]
_lib.sx_barrier_bench.argtypes = [_vp, _u32, _P(ctypes.c_double), _P(ctypes.c_int)]
_lib.sx_cluster_bench.argtypes = [_vp, _u64, _u32, _u32, _P(ctypes.c_double)]
_lib.sx_launch_bench.argtypes = [_vp, _u32, _u32, _P(ctypes.c_double)]
_lib.sx_nccl_unique_id.argtypes = [_vp]
_lib.sx_dist_create.argtypes = [_vp, _u64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _P(_vp)]
_lib.sx_dist_range.argtypes = [_vp, ctypes.c_int, _P(_u64), _P(_u64)]
_lib.sx_dist_upload.argtypes = [_vp, ctypes.c_int, _P(sx_csr_desc)]
_lib.sx_dist_free.argtypes = [_vp]
_lib.sx_dist_free.restype = None
_lib.sx_dist_bfs.argtypes = [_vp, _u32, _P(sx_opts), _P(_vp), _P(sx_stats)]
_lib.sx_dist_sssp.argtypes = [_vp, _u32, _u32, _P(sx_opts), _P(_vp), _P(sx_stats)]
_lib.sx_dist_bfs_async.argtypes = [_vp, _u32, _P(sx_opts), _P(_vp)]
_lib.sx_dist_sync.argtypes = [_vp, _P(sx_stats)]
for _f in ("sx_ctx_create", "sx_ctx_info", "sx_graph_upload", "sx_graph_info", "sx_graph_rmat", "sx_graph_grid",
           "sx_graph_download", "sx_bfs", "sx_bfs_async", "sx_graph_sync", "sx_barrier_fault", "sx_sssp",
           "sx_pagerank", "sx_pagerank_conv", "sx_bp_conv",
           "sx_kcore", "sx_spmv", "sx_bp", "sx_wcc", "sx_barrier_bench", "sx_cluster_bench", "sx_launch_bench",
           "sx_nccl_unique_id", "sx_dist_create", "sx_dist_range", "sx_dist_upload", "sx_dist_bfs", "sx_dist_sssp",
           "sx_dist_bfs_async", "sx_dist_sync"):
    getattr(_lib, _f).restype = ctypes.c_int

EXPORTED = ["sx_status_str", "sx_last_error", "sx_version", "sx_ctx_create", "sx_ctx_destroy", "sx_ctx_info",
            "sx_graph_upload", "sx_graph_info", "sx_graph_free", "sx_graph_rmat", "sx_graph_grid", "sx_graph_download",
            "sx_opts_default", "sx_bfs", "sx_bfs_async", "sx_graph_sync", "sx_barrier_fault", "sx_sssp",
            "sx_pagerank", "sx_pagerank_conv", "sx_bp_conv", "sx_kcore", "sx_spmv", "sx_bp", "sx_wcc", "sx_barrier_bench", "sx_cluster_bench", "sx_launch_bench",
            "sx_nccl_unique_id", "sx_dist_create", "sx_dist_range", "sx_dist_upload", "sx_dist_free", "sx_dist_bfs", "sx_dist_sssp",
            "sx_dist_bfs_async", "sx_dist_sync"]


class SimdxError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = _lib.sx_last_error().decode()
        super().__init__(f"{where}: {_lib.sx_status_str(status).decode()} — {detail}")


def _check(rc: int, where: str):
    if rc != SX_OK:
        raise SimdxError(rc, where)


# ---------------------------------------------------------------- pointer helpers
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if _is_torch(x):
        if not x.is_contiguous():
            raise ValueError("tensors passed to the C ABI must be contiguous")
        return x.data_ptr()
    if not (isinstance(x, np.ndarray) and x.flags["C_CONTIGUOUS"]):
        raise ValueError("host arrays must be C-contiguous numpy arrays")
    return x.ctypes.data


def _ptr_n(x, n: int, what: str) -> Optional[int]:
    """Pointer to a caller array the C side reads or writes n 4-byte elements of:
    checked for length and element size (the C ABI cannot see either)."""
    if x is None:
        return None
    size = x.numel() if _is_torch(x) else getattr(x, "size", None)
    item = x.element_size() if _is_torch(x) else getattr(getattr(x, "dtype", None), "itemsize", None)
    if item != 4:
        raise ValueError(f"{what}: 4-byte elements required (got itemsize {item})")
    if size is None or size < n:
        raise ValueError(f"{what}: {n} elements required (got {size})")
    return _ptr(x)


def _on_device(x) -> bool:
    return _is_torch(x) and x.is_cuda


# ---------------------------------------------------------------- C-named wrappers
def sx_version() -> int:
    return _lib.sx_version()


def sx_status_str(s: int) -> str:
    return _lib.sx_status_str(s).decode()


def sx_last_error() -> str:
    return _lib.sx_last_error().decode()


def sx_opts_default() -> sx_opts:
    o = sx_opts()
    _lib.sx_opts_default(ctypes.byref(o))
    return o


def make_opts(**kw) -> sx_opts:
    o = sx_opts_default()
    for k, v in kw.items():
        if k == "trace":
            continue
        setattr(o, k, v)
    return o


def sx_ctx_create(device: int = 0, stream: int = 0):
    h = _vp()
    _check(_lib.sx_ctx_create(device, _vp(stream) if stream else None, ctypes.byref(h)), "sx_ctx_create")
    return h


def sx_ctx_destroy(ctx) -> None:
    _lib.sx_ctx_destroy(ctx)


def sx_ctx_info(ctx) -> dict:
    info = sx_device_info()
    _check(_lib.sx_ctx_info(ctx, ctypes.byref(info)), "sx_ctx_info")
    return {k: getattr(info, k) for k, _ in info._fields_}


def sx_cluster_bench(ctx, nwords: int, mode: int, reps: int = 100) -> float:
    us = ctypes.c_double()
    _check(_lib.sx_cluster_bench(ctx, nwords, mode, reps, ctypes.byref(us)), "sx_cluster_bench")
    return us.value


def sx_launch_bench(ctx, mode: int, reps: int = 200) -> float:
    us = ctypes.c_double()
    _check(_lib.sx_launch_bench(ctx, mode, reps, ctypes.byref(us)), "sx_launch_bench")
    return us.value


def sx_barrier_bench(ctx, iters: int = 10000):
    us, ctas = ctypes.c_double(), ctypes.c_int()
    _check(_lib.sx_barrier_bench(ctx, iters, ctypes.byref(us), ctypes.byref(ctas)), "sx_barrier_bench")
    return us.value, ctas.value


def sx_graph_upload(ctx, n, row_ptr, col, w=None, csc_ptr=None, csc_idx=None, csc_w=None, directed=False,
                    borrow=False, dedup=False):
    """row_ptr u64[n+1], col u32[m], w u8/u32[m] or None — numpy (host) or torch CUDA tensors (device)."""
    dev = _on_device(row_ptr)
    d = sx_csr_desc()
    d.n = n
    d.m = int(row_ptr[-1])
    d.row_ptr, d.col, d.w = _ptr(row_ptr), _ptr(col), _ptr(w)
    d.w_bytes = 0 if w is None else w.element_size() if _is_torch(w) else w.dtype.itemsize
    d.csc_ptr, d.csc_idx, d.csc_w = _ptr(csc_ptr), _ptr(csc_idx), _ptr(csc_w)
    d.flags = (SX_DIRECTED if directed else 0) | (SX_DEVICE_PTRS if dev else 0) | (SX_BORROW if borrow else 0) | \
        (SX_DEDUP if dedup else 0)
    h = _vp()
    _check(_lib.sx_graph_upload(ctx, ctypes.byref(d), ctypes.byref(h)), "sx_graph_upload")
    return h


SX_GEN_NO_RELABEL = 1


def sx_graph_rmat(ctx, scale, edgefactor=16, seed=1, wmin=0, wmax=0, flags=0):
    h = _vp()
    _check(_lib.sx_graph_rmat(ctx, scale, edgefactor, seed, wmin, wmax, flags, ctypes.byref(h)), "sx_graph_rmat")
    return h


def sx_graph_grid(ctx, rows, cols, seed=1, wmin=1, wmax=255):
    h = _vp()
    _check(_lib.sx_graph_grid(ctx, rows, cols, seed, wmin, wmax, ctypes.byref(h)), "sx_graph_grid")
    return h


def sx_graph_download(g, row_ptr, col, w=None):
    """Fill caller arrays (numpy host or torch CUDA): row_ptr u64[n+1], col u32[m], w u32[m] or None."""
    _check(_lib.sx_graph_download(g, _ptr(row_ptr), _ptr(col), _ptr(w)), "sx_graph_download")


def sx_graph_free(g) -> None:
    _lib.sx_graph_free(g)


def sx_graph_info(g):
    a, b, c, d = _u64(), _u64(), _u64(), _u64()
    _check(_lib.sx_graph_info(g, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d)),
           "sx_graph_info")
    return a.value, b.value, c.value, d.value


def _nv(g, n):
    """Vertex count of g's output arrays (this rank's slice); n given by the caller skips the query."""
    if n is not None:
        return n
    a, _, lo, hi = sx_graph_info(g)
    return hi - lo


def _run(fn, name, g, out, opts, args_before, args_after=(), n=None):
    st = sx_stats()
    o = opts if opts is not None else sx_opts_default()
    _check(fn(g, *args_before, ctypes.byref(o), *args_after, _ptr_n(out, _nv(g, n), name + " out"),
              ctypes.byref(st)), name)
    return st


def sx_bfs(g, src, opts, level_out, n=None):
    return _run(_lib.sx_bfs, "sx_bfs", g, level_out, opts, (src,), n=n)


def sx_bfs_async(g, src, opts, level_out, n=None):
    """Enqueue a BFS (all fusion) without waiting; level_out must be a CUDA tensor."""
    if not _on_device(level_out):
        raise ValueError("sx_bfs_async: level_out must be a CUDA tensor")
    o = opts if opts is not None else sx_opts_default()
    _check(_lib.sx_bfs_async(g, src, ctypes.byref(o), _ptr_n(level_out, _nv(g, n), "sx_bfs_async out")),
           "sx_bfs_async")


def sx_graph_sync(g) -> sx_stats:
    st = sx_stats()
    _check(_lib.sx_graph_sync(g, ctypes.byref(st)), "sx_graph_sync")
    return st


def sx_barrier_fault(ctx, mode: int, timeout_ms: int = 0) -> int:
    """Status code of the injected barrier fault (SX_E_BARRIER = detected)."""
    return _lib.sx_barrier_fault(ctx, mode, timeout_ms)


def sx_sssp(g, src, delta, opts, dist_out, n=None):
    return _run(_lib.sx_sssp, "sx_sssp", g, dist_out, opts, (src, delta), n=n)


def sx_pagerank(g, damping, iters, opts, rank_out, n=None):
    return _run(_lib.sx_pagerank, "sx_pagerank", g, rank_out, opts, (damping, iters), n=n)


SX_PR_NORMALIZED, SX_PR_SPEC = 0, 1


def sx_pagerank_conv(g, damping, epsilon, max_iters, variant, opts, rank_out, n=None):
    n = _nv(g, n)
    if rank_out is not None and (rank_out.element_size() if _is_torch(rank_out) else rank_out.dtype.itemsize) != 8:
        raise ValueError("sx_pagerank_conv out: 8-byte (float64) elements required")
    st = sx_stats()
    o = opts if opts is not None else sx_opts_default()
    size = rank_out.numel() if _is_torch(rank_out) else rank_out.size
    if size < n:
        raise ValueError(f"sx_pagerank_conv out: {n} elements required (got {size})")
    _check(_lib.sx_pagerank_conv(g, damping, epsilon, max_iters, variant, ctypes.byref(o), _ptr(rank_out),
                                 ctypes.byref(st)), "sx_pagerank_conv")
    return st


def sx_bp_conv(g, prior, epsilon, max_iters, opts, out, n=None):
    n = _nv(g, n)
    return _run(_lib.sx_bp_conv, "sx_bp_conv", g, out, opts, (_ptr_n(prior, n, "sx_bp_conv prior"), epsilon, max_iters),
                n=n)


def sx_kcore(g, k, opts, core_out, n=None):
    return _run(_lib.sx_kcore, "sx_kcore", g, core_out, opts, (k,), n=n)


def sx_spmv(g, x, iters, opts, y_out, n=None):
    n = _nv(g, n)
    return _run(_lib.sx_spmv, "sx_spmv", g, y_out, opts, (_ptr_n(x, n, "sx_spmv x"), iters), n=n)


def sx_wcc(g, opts, label_out, n=None):
    return _run(_lib.sx_wcc, "sx_wcc", g, label_out, opts, (), n=n)


def sx_bp(g, prior, iters, opts, out, n=None):
    n = _nv(g, n)
    return _run(_lib.sx_bp, "sx_bp", g, out, opts, (_ptr_n(prior, n, "sx_bp prior"), iters), n=n)


# ---------------------------------------------------------------- conveniences
class Context:
    def __init__(self, device: int = 0, stream: int = 0):
        self.h = sx_ctx_create(device, stream)

    def info(self) -> dict:
        return sx_ctx_info(self.h)

    def upload_device(self, dcsr, borrow: bool = False) -> "Graph":
        """Upload from raw device pointers (e.g. simgen.DeviceCSR); borrow = no copy."""
        d = sx_csr_desc()
        d.n, d.m = dcsr.v_hi - dcsr.v_lo, dcsr.m
        d.row_ptr, d.col, d.w = dcsr.row_ptr_ptr, dcsr.col_ptr, dcsr.w_ptr
        d.w_bytes = dcsr.wbytes
        d.flags = SX_DEVICE_PTRS | (SX_BORROW if borrow else 0)
        h = _vp()
        _check(_lib.sx_graph_upload(self.h, ctypes.byref(d), ctypes.byref(h)), "sx_graph_upload")
        return Graph(self, h, d.n)

    def rmat(self, scale: int, edgefactor: int = 16, seed: int = 1, wmin: int = 0, wmax: int = 0,
             relabel: bool = True) -> "Graph":
        """sx_graph_rmat: the simgen R-MAT graph built on the device (bit-identical to simgen.rmat)."""
        h = sx_graph_rmat(self.h, scale, edgefactor, seed, wmin, wmax, 0 if relabel else SX_GEN_NO_RELABEL)
        return Graph(self, h, 1 << scale)

    def grid(self, rows: int, cols: int, seed: int = 1, wmin: int = 1, wmax: int = 255) -> "Graph":
        """sx_graph_grid: the simgen rows x cols grid built on the device."""
        return Graph(self, sx_graph_grid(self.h, rows, cols, seed, wmin, wmax), rows * cols)

    def upload(self, csr, dedup: bool = False) -> "Graph":
        """Upload a simgen.CSR-like object (fields n,row_ptr,col,w,directed,csc_*); dedup: SX_DEDUP."""
        h = sx_graph_upload(self.h, csr.n, csr.row_ptr, csr.col, csr.w,
                            getattr(csr, "csc_ptr", None), getattr(csr, "csc_idx", None),
                            getattr(csr, "csc_w", None), bool(getattr(csr, "directed", False)), dedup=dedup)
        return Graph(self, h, csr.n)

    def close(self):
        if self.h:
            sx_ctx_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Graph:
    def __init__(self, ctx: Context, h, n: int):
        self.ctx, self.h, self.n = ctx, h, n

    def info(self):
        """(n, m, v_begin, v_end)"""
        return sx_graph_info(self.h)

    def download(self, weights: bool = True):
        """Host copy of the CSR: (row_ptr u64[n+1], col u32[m], w u32[m] or None)."""
        n, m, _, _ = sx_graph_info(self.h)
        rp = np.empty(n + 1, np.uint64)
        col = np.empty(m, np.uint32)
        w = np.empty(m, np.uint32) if weights else None
        sx_graph_download(self.h, rp, col, w)
        return rp, col, w

    def free(self):
        if self.h:
            sx_graph_free(self.h)
            self.h = None

    _default_opts = None

    _opts_cache: dict = {}

    def _opts(self, kw):
        if not kw:  # the common call: default options, built once
            if Graph._default_opts is None:
                Graph._default_opts = make_opts()
            return Graph._default_opts, None
        if "trace_cap" not in kw:  # repeated option sets without a trace: built once each
            key = tuple(sorted(kw.items()))
            o = Graph._opts_cache.get(key)
            if o is None:
                o = Graph._opts_cache[key] = make_opts(**kw)
            return o, None
        trace_cap = kw.pop("trace_cap", 0)
        o = make_opts(**kw)
        buf = None
        if trace_cap:
            buf = (sx_trace_rec * trace_cap)()
            o.trace = ctypes.cast(buf, ctypes.POINTER(sx_trace_rec))
            o.trace_cap = trace_cap
        return o, buf

    @staticmethod
    def _trace(buf, st):
        if buf is None:
            return None
        recs = []
        for r in buf:
            if r.t_ns == 0:
                break
            recs.append(dict(iter=r.iter, dir=r.dir, filter=r.filter, launch=r.launch, n_active=list(r.n_active),
                             n_frontier=r.n_frontier, m_active=r.m_active, aux=r.aux, t_ns=r.t_ns))
        return recs

    def bfs(self, src: int, out=None, **kw):
        out = np.empty(self.n, np.uint32) if out is None else out
        o, buf = self._opts(dict(kw))
        st = sx_bfs(self.h, src, o, out, self.n)
        return out, st.as_dict(), self._trace(buf, st)

    def bfs_async(self, src: int, out, **kw):
        """sx_bfs_async: enqueue one BFS into the CUDA tensor `out`; no wait."""
        o, _ = self._opts(dict(kw))
        sx_bfs_async(self.h, src, o, out, self.n)

    def sync(self) -> dict:
        """sx_graph_sync: wait for the enqueued runs; their summed statistics."""
        return sx_graph_sync(self.h).as_dict()

    def sssp(self, src: int, delta: int = 0, out=None, **kw):
        out = np.empty(self.n, np.uint32) if out is None else out
        o, buf = self._opts(dict(kw))
        st = sx_sssp(self.h, src, delta, o, out, self.n)
        return out, st.as_dict(), self._trace(buf, st)

    def pagerank(self, damping: float = 0.85, iters: int = 20, out=None, **kw):
        out = np.empty(self.n, np.float32) if out is None else out
        o, buf = self._opts(dict(kw))
        st = sx_pagerank(self.h, damping, iters, o, out, self.n)
        return out, st.as_dict(), self._trace(buf, st)

    def pagerank_conv(self, damping: float = 0.85, eps: float = 1e-6, max_iters: int = 10000, variant: int = 0,
                      out=None, **kw):
        out = np.empty(self.n, np.float64) if out is None else out
        o, buf = self._opts(dict(kw))
        st = sx_pagerank_conv(self.h, damping, eps, max_iters, variant, o, out, self.n)
        return out, st.as_dict(), self._trace(buf, st)

    def bp_conv(self, prior, eps: float = 1e-6, max_iters: int = 1000, out=None, **kw):
        out = np.empty(self.n, np.float32) if out is None else out
        o, buf = self._opts(dict(kw))
        st = sx_bp_conv(self.h, prior, eps, max_iters, o, out, self.n)
        return out, st.as_dict(), self._trace(buf, st)

    def kcore(self, k: int = 0, out=None, **kw):
        out = np.empty(self.n, np.uint32) if out is None else out
        o, buf = self._opts(dict(kw))
        st = sx_kcore(self.h, k, o, out, self.n)
        return out, st.as_dict(), self._trace(buf, st)

    def wcc(self, out=None, **kw):
        out = np.empty(self.n, np.uint32) if out is None else out
        o, buf = self._opts(dict(kw))
        st = sx_wcc(self.h, o, out, self.n)
        return out, st.as_dict(), self._trace(buf, st)

    def spmv(self, x, iters: int = 1, out=None, **kw):
        out = np.empty(self.n, np.float32) if out is None else out
        o, buf = self._opts(dict(kw))
        st = sx_spmv(self.h, x, iters, o, out, self.n)
        return out, st.as_dict(), self._trace(buf, st)

    def bp(self, prior, iters: int = 10, out=None, **kw):
        out = np.empty(self.n, np.float32) if out is None else out
        o, buf = self._opts(dict(kw))
        st = sx_bp(self.h, prior, iters, o, out, self.n)
        return out, st.as_dict(), self._trace(buf, st)


# ---------------------------------------------------------------- multi-GPU layer
def sx_nccl_unique_id() -> bytes:
    buf = (ctypes.c_char * 128)()
    _check(_lib.sx_nccl_unique_id(buf), "sx_nccl_unique_id")
    return bytes(buf)


def partition(n: int, nranks: int, rank: int):
    """Owned vertex range of `rank` (the rule of sx_dist_create: V = ceil(n/P) rounded up to 32)."""
    V = ((n + nranks - 1) // nranks + 31) // 32 * 32 or 32
    lo = min(n, rank * V)
    return lo, min(n, lo + V)


class Dist:
    """A graph distributed by 1D vertex ranges.

    nlocal == nranks: all ranks in this process on one device (virtual ranks);
    nlocal == 1: this process is rank `rank0` of an NCCL job (`nccl_id` from rank 0).
    """

    def __init__(self, ctx: Context, n: int, nranks: int, rank0: int = 0, nlocal: Optional[int] = None,
                 nccl_id: Optional[bytes] = None):
        nlocal = nranks if nlocal is None else nlocal
        self.ctx, self.n, self.nranks, self.rank0, self.nlocal = ctx, n, nranks, rank0, nlocal
        h = _vp()
        idbuf = None if nccl_id is None else ctypes.create_string_buffer(nccl_id, 128)
        _check(_lib.sx_dist_create(ctx.h, n, nranks, rank0, nlocal, idbuf, ctypes.byref(h)), "sx_dist_create")
        self.h = h

    def range(self, local_rank: int):
        a, b = _u64(), _u64()
        _check(_lib.sx_dist_range(self.h, local_rank, ctypes.byref(a), ctypes.byref(b)), "sx_dist_range")
        return a.value, b.value

    def upload_device(self, local_rank: int, dcsr) -> None:
        """Upload a rank's slice from raw device pointers (simgen.DeviceCSR with v_lo/v_hi)."""
        d = sx_csr_desc()
        d.n, d.m = dcsr.v_hi - dcsr.v_lo, dcsr.m
        d.row_ptr, d.col, d.w = dcsr.row_ptr_ptr, dcsr.col_ptr, dcsr.w_ptr
        d.w_bytes = dcsr.wbytes
        d.flags = SX_DEVICE_PTRS
        _check(_lib.sx_dist_upload(self.h, local_rank, ctypes.byref(d)), "sx_dist_upload")

    def upload(self, local_rank: int, csr_slice) -> None:
        """csr_slice: rows [v_lo, v_hi) (simgen.CSR with v_lo/v_hi), global column ids."""
        d = sx_csr_desc()
        d.n = int(csr_slice.row_ptr.shape[0] - 1)
        d.m = int(csr_slice.row_ptr[-1])
        d.row_ptr, d.col, d.w = _ptr(csr_slice.row_ptr), _ptr(csr_slice.col), _ptr(csr_slice.w)
        d.w_bytes = 0 if csr_slice.w is None else csr_slice.w.dtype.itemsize
        d.flags = 0
        _check(_lib.sx_dist_upload(self.h, local_rank, ctypes.byref(d)), "sx_dist_upload")

    def _outs(self, outs):
        if outs is None:
            outs = []
            for i in range(self.nlocal):
                lo, hi = self.range(i)
                outs.append(np.empty(hi - lo, np.uint32))
        if len(outs) != self.nlocal:
            raise ValueError(f"Dist: {self.nlocal} output slices required (got {len(outs)})")
        ptrs = []
        for i, o in enumerate(outs):
            lo, hi = self.range(i)
            ptrs.append(_ptr_n(o, hi - lo, f"Dist output slice {i}"))
        arr = (_vp * self.nlocal)(*ptrs)
        return outs, arr

    def bfs(self, src: int, outs=None, **kw):
        outs, arr = self._outs(outs)
        st = sx_stats()
        o = make_opts(**kw)
        _check(_lib.sx_dist_bfs(self.h, src, ctypes.byref(o), arr, ctypes.byref(st)), "sx_dist_bfs")
        return outs, st.as_dict()

    def bfs_async(self, src: int, outs, **kw):
        """Enqueue a device-initiated BFS (sx_dist_bfs_async); outs: device tensors (owned slice)."""
        outs, arr = self._outs(outs)
        o = make_opts(**kw)
        _check(_lib.sx_dist_bfs_async(self.h, src, ctypes.byref(o), arr), "sx_dist_bfs_async")
        return outs

    def sync(self):
        """Wait for the async runs (sx_dist_sync); their statistics."""
        st = sx_stats()
        _check(_lib.sx_dist_sync(self.h, ctypes.byref(st)), "sx_dist_sync")
        return st.as_dict()

    def sssp(self, src: int, delta: int = 0, outs=None, **kw):
        outs, arr = self._outs(outs)
        st = sx_stats()
        o = make_opts(**kw)
        _check(_lib.sx_dist_sssp(self.h, src, delta, ctypes.byref(o), arr, ctypes.byref(st)), "sx_dist_sssp")
        return outs, st.as_dict()

    def free(self):
        if self.h:
            _lib.sx_dist_free(self.h)
            self.h = None
