"""CPU-side checks of the boundary: libtango.so builds for sm_100a, loads without a GPU,
and exports every entry point include/tango.h declares; host-side validation errors
are returned synchronously (no device needed for those paths)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2308_00890_b200 import build, tango
    build.build()
    return tango.load()


def declared():
    src = open(os.path.join(ROOT, "include", "tango.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tango_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    names = declared()
    for need in ["tango_quantize", "tango_gemm_q", "tango_sddmm_q", "tango_spmm_q", "tango_gat_layer_fwd",
                 "tango_gat_layer_bwd", "tango_gcn_layer_fwd", "tango_gcn_layer_bwd"]:
        assert need in names


def test_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_lists_every_export(lib):
    from paper_2308_00890_b200 import tango
    assert sorted(tango.EXPORTS) == declared()


def test_sass_is_sm100a_with_tcgen05(lib):
    from paper_2308_00890_b200 import tango
    out = subprocess.run(["cuobjdump", "-sass", tango.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCQMMA" in out or "UTCIMMA" in out or re.search(r"UTC\w*MMA", out)   # tcgen05.mma
    assert "UTMALDG" in out                                                           # TMA loads
    assert "IDP.4A" in out                                                            # SDDMM-dot on codes


def test_status_strings_and_validation_without_gpu(lib):
    lib.tango_status_string.restype = C.c_char_p
    assert lib.tango_status_string(0) == b"ok"
    assert lib.tango_abi_version() == 1
    from paper_2308_00890_b200 import tango as T
    # NULL graph -> INVALID_ARG, bad bits -> BITS: returned before any CUDA call
    p = T.GatParams(None, None, None, 16, 2, 32, 0.2, 8)
    assert lib.tango_gat_ctx_bytes(None, C.byref(p)) == 0
    g = T.Graph(10, 0, 10, 1, 1, 0, 1, 1, None, 0, 256)   # fake non-NULL pointers: validation only
    p = T.GatParams(1, 1, 1, 16, 3, 16, 0.2, 8)           # HD = 48 unsupported
    assert lib.tango_gat_ctx_bytes(C.byref(g), C.byref(p)) == 0
    p = T.GatParams(1, 1, 1, 16, 2, 32, 0.2, 8)
    assert lib.tango_gat_ctx_bytes(C.byref(g), C.byref(p)) > 0
    q = T.QTensor(1, 1, 4, 4, 16, 9)
    st = lib.tango_gemm_q(C.byref(q), 0, C.byref(q), 0, 4, 4, 4, 1, None, None, None)
    assert st == 3   # TANGO_ERR_BITS


def test_no_cpu_fallback(tmp_path):
    from paper_2308_00890_b200 import tango
    saved = tango._lib
    tango._lib = None
    try:
        with pytest.raises(ImportError):
            tango.load(str(tmp_path / "missing.so"))
    finally:
        tango._lib = saved


def test_next_entry_points_validate_without_gpu(lib):
    """Host-side argument validation of the NEXT-1 / NEXT-4 entry points returns before any CUDA call."""
    from paper_2308_00890_b200 import tango as T
    # tango_sgemm: bad layout -> INVALID_ARG, negative size -> SHAPE, missing workspace for K > 1024 -> INVALID_ARG
    assert lib.tango_sgemm(1, 4, 7, 1, 4, 0, 4, 4, 4, 1, None, 0, None) == 1
    assert lib.tango_sgemm(1, 4, 0, 1, 4, 0, -1, 4, 4, 1, None, 0, None) == 2
    assert lib.tango_sgemm_workspace_bytes(64, 64, 1024) == 0
    assert lib.tango_sgemm_workspace_bytes(64, 64, 1025) == 2 * 64 * 64 * 4
    assert lib.tango_sgemm(1, 2048, 0, 1, 64, 1, 64, 64, 2048, 1, None, 0, None) == 1
    # cross-entropy: classes > 1024 -> UNSUPPORTED, n_labeled > rows -> SHAPE
    assert lib.tango_cross_entropy(1, 1, 10, 2000, 5, 1, 1, None, None) == 6
    assert lib.tango_cross_entropy(1, 1, 10, 7, 11, 1, 1, None, None) == 2
    # sgd: more than 32 tensors -> UNSUPPORTED
    assert lib.tango_sgd_update(None, 33, 0.1, None) == 6
    # FP32 final layers are one-GPU only: a partitioned graph view has no ctx size
    g = T.Graph(100, 0, 50, 1, 1, 10, 1, 1, 1, 10, 256)
    p = T.GatOutParams(1, 1, 1, 1, 16, 4, 40, 0.2)
    assert lib.tango_gat_out_ctx_bytes(C.byref(g), C.byref(p)) == 0
    g.row_end = 100
    assert lib.tango_gat_out_ctx_bytes(C.byref(g), C.byref(p)) > 0
    p.heads, p.classes = 8, 200                                   # H*C > 1024
    assert lib.tango_gat_out_ctx_bytes(C.byref(g), C.byref(p)) == 0
    gp = T.GcnOutParams(1, 1, 16, 7)
    assert lib.tango_gcn_out_ctx_bytes(C.byref(g), C.byref(gp)) > 0
    # INT4: cols not a multiple of 8 -> SHAPE; bits other than 4 / 8 -> BITS
    assert lib.tango_quantize_int4(1, 4, 12, 0, None, T.Rng(0, 0, 0), 16, 8, 1, 1, None, None) == 2
    assert lib.tango_sddmm_qn(C.byref(g), 1, 5, 16, 16, 16, 16, 16, 16, 4, 64, 0.2, 16, None, None) == 3
