"""The C-ABI library loads and exports every symbol include/simdx.h declares
(no compute calls: this runs on the CPU-only box too)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "simdx.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(sx_[a-z_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("sx_ctx_create", "sx_graph_upload", "sx_bfs", "sx_sssp", "sx_pagerank", "sx_kcore", "sx_spmv",
                 "sx_bp", "sx_graph_free", "sx_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1812_04070_b200 import simdx
    lib = ctypes.CDLL(simdx.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(simdx.EXPORTED) == declared_functions()


def test_library_is_sm100a_only():
    import subprocess
    from paper_1812_04070_b200 import simdx
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", simdx.LIB_PATH], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_status_strings_and_version():
    from paper_1812_04070_b200 import simdx
    assert simdx.sx_status_str(0) == "SX_OK"
    assert simdx.sx_status_str(7) == "SX_E_BARRIER"
    assert simdx.sx_status_str(99) == "SX_E_UNKNOWN"
    assert simdx.sx_version() >= 1
    o = simdx.sx_opts_default()
    assert (o.overflow_threshold, o.sep_small, o.sep_large) == (64, 32, 128)
    assert o.fusion == 1 and o.force_filter == 0 and o.force_dir == 0
    assert o.cluster_enter == 0xFFFFFFFF  # SX_CLUSTER_AUTO: resolved per algorithm and graph size


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1812_04070_b200 import simdx
    with pytest.raises(simdx.SimdxError) as e:
        simdx.sx_ctx_create(0)
    assert e.value.status == simdx.SX_E_CUDA


def test_trace_and_stats_struct_sizes():
    from paper_1812_04070_b200 import simdx
    assert ctypes.sizeof(simdx.sx_trace_rec) == 64
    assert ctypes.sizeof(simdx.sx_stats) == 4 * 4 + 3 * 8 + 6 * 8 + 2 * 4 + 8 + 2 * 4 + 8


def test_binding_checks_caller_buffers():
    """Output / input arrays are checked for length and element size before the
    C call (the C side writes n 4-byte elements and cannot see either)."""
    import numpy as np
    from paper_1812_04070_b200 import simdx
    with pytest.raises(ValueError):
        simdx.sx_bfs(None, 0, None, np.empty(3, np.uint32), n=10)
    with pytest.raises(ValueError):
        simdx.sx_sssp(None, 0, 0, None, np.empty(10, np.uint64), n=10)
    with pytest.raises(ValueError):
        simdx.sx_pagerank(None, 0.85, 20, None, np.empty((10, 2), np.float32)[:, 0], n=10)
    with pytest.raises(ValueError):
        simdx.sx_spmv(None, np.empty(9, np.float32), 1, None, np.empty(10, np.float32), n=10)
    with pytest.raises(ValueError):
        simdx.sx_bp(None, np.empty(10, np.float64), 1, None, np.empty(10, np.float32), n=10)
