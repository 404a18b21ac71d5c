"""Thin ctypes binding of libtango.so (include/tango.h).

Argument marshalling only: every step of the path runs in the library's CUDA kernels.
PyTorch provides device memory and the current CUDA stream.  There is no fallback:
if libtango.so is missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from .partition import local_graph

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtango.so")

TANGO_K_MAJOR, TANGO_MN_MAJOR = 0, 1
TANGO_SDDMM_ADD, TANGO_SDDMM_DOT = 0, 1
TANGO_IN, TANGO_OUT = 0, 1
ROLE = dict(H=1, W=2, Hp=3, S=4, D=5, G=6, dHp=7, Ys=8, Gs=9, dY=10)
STATUS = {0: "ok", 1: "invalid argument", 2: "shape mismatch", 3: "bits", 4: "non-finite", 5: "overflow",
          6: "unsupported", 7: "CUDA error", 8: "NCCL error"}


class TangoError(RuntimeError):
    def __init__(self, status, what=""):
        super().__init__(f"{what}: tango status {status} ({STATUS.get(status, '?')})")
        self.status = status


_P = C.c_void_p


class Graph(C.Structure):
    _fields_ = [("n_global", C.c_int64), ("row_begin", C.c_int64), ("row_end", C.c_int64), ("in_ptr", _P),
                ("in_src", _P), ("e_in", C.c_int64), ("out_ptr", _P), ("out_dst", _P), ("out_eid", _P),
                ("e_out", C.c_int64), ("chunk_edges", C.c_int32), ("graph_id", C.c_uint64)]


class QTensor(C.Structure):
    _fields_ = [("q", _P), ("scale", _P), ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64),
                ("bits", C.c_int32)]


class Rng(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("step", C.c_uint32), ("tag", C.c_uint32)]


class GatParams(C.Structure):
    _fields_ = [("W", _P), ("a_src", _P), ("a_dst", _P), ("in_feats", C.c_int32), ("heads", C.c_int32),
                ("head_dim", C.c_int32), ("neg_slope", C.c_float), ("bits", C.c_int32)]


class GatCtxView(C.Structure):
    _fields_ = [(f, _P) for f in ("qH", "qW", "qWt", "qHp", "qS", "qD", "qG", "qdHp")] + \
               [(f, C.c_int64) for f in ("ldF", "ldHD", "ldFt")] + \
               [(f, _P) for f in ("S", "D", "m", "den", "P", "dD", "dHp", "dalpha", "alpha_pack", "scalars")] + \
               [("codes_biased", C.c_int32), ("dS", _P), ("dataflow", C.c_int32)]


class GcnParams(C.Structure):
    _fields_ = [("W", _P), ("in_feats", C.c_int32), ("out_feats", C.c_int32), ("bits", C.c_int32)]


class GcnCtxView(C.Structure):
    _fields_ = [(f, _P) for f in ("qX", "qW", "qWt", "qYs", "qGs", "qdY")] + \
               [(f, C.c_int64) for f in ("ldF", "ldO", "ldFt")] + [(f, _P) for f in ("ia", "ib", "scalars")]


class GatOutParams(C.Structure):
    _fields_ = [("W", _P), ("a_src", _P), ("a_dst", _P), ("bias", _P), ("in_feats", C.c_int32),
                ("heads", C.c_int32), ("classes", C.c_int32), ("neg_slope", C.c_float)]


_OUT_VIEW = ("Hp", "S", "D", "e_pre", "alpha", "m", "den", "G", "dalpha", "dE_pre", "P", "dD", "dS", "dHp", "agg")


class GatOutCtxView(C.Structure):
    _fields_ = [(f, _P) for f in _OUT_VIEW]


class GcnOutParams(C.Structure):
    _fields_ = [("W", _P), ("bias", _P), ("in_feats", C.c_int32), ("classes", C.c_int32)]


class GcnOutCtxView(C.Structure):
    _fields_ = [(f, _P) for f in ("Y", "Ys", "agg", "Gs", "aggb", "dY")]


class SgdTensor(C.Structure):
    _fields_ = [("w", _P), ("g", _P), ("count", C.c_int64)]


_lib = None

EXPORTS = ["tango_status_string", "tango_abi_version", "tango_status_poll", "tango_quantize", "tango_gemm_q",
           "tango_sddmm_q", "tango_edge_softmax", "tango_softmax_bwd", "tango_spmm_q", "tango_edge_sum",
           "tango_gat_ctx_bytes", "tango_gat_layer_fwd", "tango_gat_layer_bwd", "tango_gat_ctx_get_view",
           "tango_gcn_ctx_bytes", "tango_gcn_layer_fwd", "tango_gcn_layer_bwd", "tango_gcn_ctx_get_view",
           "tango_comm_unique_id_bytes", "tango_comm_get_unique_id", "tango_comm_init", "tango_comm_destroy",
           "tango_comm_set_partition", "tango_local_group_create", "tango_local_group_destroy",
           "tango_comm_init_local", "tango_quant_error", "tango_select_bits", "tango_profile_enable", "tango_launch_count", "tango_profile_collect",
           "tango_profile_num_entries", "tango_profile_entry", "tango_profile_reset", "tango_profile_serialize",
           "tango_sgemm_workspace_bytes", "tango_sgemm", "tango_colsum_workspace_bytes", "tango_colsum",
           "tango_bias_act_fwd", "tango_bias_act_bwd", "tango_cross_entropy", "tango_sgd_update",
           "tango_gat_out_ctx_bytes", "tango_gat_out_fwd", "tango_gat_out_bwd", "tango_gat_out_ctx_get_view",
           "tango_gcn_out_ctx_bytes", "tango_gcn_out_fwd", "tango_gcn_out_bwd", "tango_gcn_out_ctx_get_view",
           "tango_quantize_int4", "tango_sddmm_qn", "tango_set_l2_fetch_granularity", "tango_comm_set_options",
           "tango_comm_reserve", "tango_comm_nccl_calls", "tango_spmm_q8", "tango_nvtx_enable"]


def load(path: str = LIB_PATH):
    """Load libtango.so (no compute call; works without a GPU)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_2308_00890_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(path)
    i32, i64, u32, f32, sz = C.c_int32, C.c_int64, C.c_uint32, C.c_float, C.c_size_t
    PG, PQ = C.POINTER(Graph), C.POINTER(QTensor)
    L.tango_status_string.restype = C.c_char_p
    L.tango_status_string.argtypes = [C.c_int]
    L.tango_status_poll.argtypes = [_P, _P, C.POINTER(C.c_int)]
    L.tango_quantize.argtypes = [_P, i64, i64, i64, _P, Rng, PQ, _P, _P, _P]
    L.tango_gemm_q.argtypes = [PQ, i32, PQ, i32, i64, i64, i64, _P, _P, _P, _P]
    L.tango_sddmm_q.argtypes = [PG, i32, PQ, PQ, i32, f32, _P, _P, _P, _P]
    L.tango_edge_softmax.argtypes = [PG, i32, _P, _P, _P, _P, _P]
    L.tango_softmax_bwd.argtypes = [PG, i32, _P, _P, _P, f32, _P, _P, _P]
    L.tango_spmm_q.argtypes = [PG, i32, _P, PQ, i32, _P, _P, _P, _P, _P]
    L.tango_edge_sum.argtypes = [PG, i32, i32, _P, _P, _P]
    L.tango_set_l2_fetch_granularity.argtypes = [i32, _P]
    L.tango_comm_set_options.argtypes = [_P, i32]
    L.tango_comm_reserve.argtypes = [_P, sz]
    L.tango_comm_nccl_calls.argtypes = [_P]
    L.tango_spmm_q8.argtypes = [PG, i32, PQ, PQ, i32, _P, _P, _P]
    L.tango_nvtx_enable.argtypes = [i32]
    L.tango_nvtx_enable.restype = None
    L.tango_comm_nccl_calls.restype = C.c_int64
    L.tango_gat_ctx_bytes.restype = sz
    L.tango_gat_ctx_bytes.argtypes = [PG, C.POINTER(GatParams)]
    L.tango_gat_ctx_get_view.argtypes = [PG, C.POINTER(GatParams), _P, C.POINTER(GatCtxView)]
    L.tango_gat_layer_fwd.argtypes = [PG, C.POINTER(GatParams), _P, _P, Rng, u32, _P, sz, _P, _P, _P, _P, _P]
    L.tango_gat_layer_bwd.argtypes = [PG, C.POINTER(GatParams), _P, sz, _P, _P, Rng, u32, _P, _P, _P, _P, _P, _P,
                                      _P, _P]
    L.tango_gcn_ctx_bytes.restype = sz
    L.tango_gcn_ctx_bytes.argtypes = [PG, C.POINTER(GcnParams)]
    L.tango_gcn_ctx_get_view.argtypes = [PG, C.POINTER(GcnParams), _P, C.POINTER(GcnCtxView)]
    L.tango_gcn_layer_fwd.argtypes = [PG, C.POINTER(GcnParams), _P, _P, Rng, u32, _P, sz, _P, _P, _P, _P, _P]
    L.tango_gcn_layer_bwd.argtypes = [PG, C.POINTER(GcnParams), _P, sz, _P, Rng, u32, _P, _P, _P, _P, _P]
    L.tango_comm_unique_id_bytes.restype = i32
    L.tango_comm_get_unique_id.argtypes = [_P]
    L.tango_comm_init.argtypes = [C.POINTER(_P), _P, i32, i32]
    L.tango_comm_destroy.argtypes = [_P]
    L.tango_comm_set_partition.argtypes = [_P, _P]
    L.tango_quant_error.argtypes = [_P, i64, i64, PQ, _P, _P]
    L.tango_select_bits.argtypes = [_P, i64, f32, i32, i32, _P, _P, _P]
    L.tango_local_group_create.argtypes = [C.POINTER(_P), i32]
    L.tango_local_group_destroy.argtypes = [_P]
    L.tango_comm_init_local.argtypes = [C.POINTER(_P), _P, i32]
    L.tango_profile_enable.argtypes = [i32]
    L.tango_profile_enable.restype = None
    L.tango_launch_count.restype = i64
    L.tango_profile_num_entries.restype = i32
    L.tango_profile_entry.argtypes = [i32, C.c_char_p, i32, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    L.tango_profile_reset.restype = None
    L.tango_profile_serialize.argtypes = [i32]
    L.tango_profile_serialize.restype = None
    L.tango_sgemm_workspace_bytes.restype = sz
    L.tango_sgemm_workspace_bytes.argtypes = [i64, i64, i64]
    L.tango_sgemm.argtypes = [_P, i64, i32, _P, i64, i32, i64, i64, i64, _P, _P, sz, _P]
    L.tango_colsum_workspace_bytes.restype = sz
    L.tango_colsum_workspace_bytes.argtypes = [i64, i64]
    L.tango_colsum.argtypes = [_P, i64, i64, _P, _P, sz, _P]
    L.tango_bias_act_fwd.argtypes = [_P, _P, i64, i64, _P, _P, _P]
    L.tango_bias_act_bwd.argtypes = [_P, _P, i64, i64, _P, _P, _P, _P, sz, _P]
    L.tango_cross_entropy.argtypes = [_P, _P, i64, i32, i64, _P, _P, _P, _P]
    L.tango_sgd_update.argtypes = [C.POINTER(SgdTensor), i32, f32, _P]
    PO = C.POINTER(GatOutParams)
    L.tango_gat_out_ctx_bytes.restype = sz
    L.tango_gat_out_ctx_bytes.argtypes = [PG, PO]
    L.tango_gat_out_fwd.argtypes = [PG, PO, _P, _P, sz, _P, _P]
    L.tango_gat_out_bwd.argtypes = [PG, PO, _P, sz, _P, _P, _P, _P, _P, _P, _P, _P]
    L.tango_gat_out_ctx_get_view.argtypes = [PG, PO, _P, C.POINTER(GatOutCtxView)]
    L.tango_quantize_int4.argtypes = [_P, i64, i64, i64, _P, Rng, _P, i64, _P, _P, _P, _P]
    L.tango_sddmm_qn.argtypes = [PG, i32, i32, _P, i64, _P, _P, i64, _P, i32, i32, f32, _P, _P, _P]
    PGO = C.POINTER(GcnOutParams)
    L.tango_gcn_out_ctx_bytes.restype = sz
    L.tango_gcn_out_ctx_bytes.argtypes = [PG, PGO]
    L.tango_gcn_out_fwd.argtypes = [PG, PGO, _P, _P, sz, _P, _P]
    L.tango_gcn_out_bwd.argtypes = [PG, PGO, _P, sz, _P, _P, _P, _P, _P, _P]
    L.tango_gcn_out_ctx_get_view.argtypes = [PG, PGO, _P, C.POINTER(GcnOutCtxView)]
    _lib = L
    return L


def _check(st, what):
    if st != 0:
        raise TangoError(st, what)


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise TypeError("libtango takes CUDA tensors only")
    if not t.is_contiguous():
        raise ValueError("libtango takes contiguous tensors only (row strides are passed explicitly)")
    return t.data_ptr()


def _arg(t, name, shape, dtype=torch.float32, optional=False):
    """Pointer of a layer argument after checking what the C ABI assumes of it: a contiguous CUDA tensor
    of the given dtype and shape (a transposed, sliced or mistyped tensor would be read with the wrong
    layout without an error)."""
    if t is None:
        if optional:
            return None
        raise ValueError(f"{name}: required")
    if t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    return _ptr(t)


def _stream():
    return torch.cuda.current_stream().cuda_stream


def ld32(cols: int) -> int:
    return (cols + 31) // 32 * 32


# ---------------------------------------------------------------------------------------- tracing
def profile_enable(on: bool = True):
    load().tango_profile_enable(1 if on else 0)


def nvtx_enable(on: bool = True):
    """NVTX range per library kernel launch (timeline tools); also TANGO_NVTX=1."""
    load().tango_nvtx_enable(1 if on else 0)


def profile_serialize(on: bool = True):
    """Side-stream work in order on the caller's stream (per-kernel event times without overlap)."""
    load().tango_profile_serialize(1 if on else 0)


def set_l2_fetch_granularity(nbytes: int) -> int:
    """cudaLimitMaxL2FetchGranularity for the current device (tango_set_l2_fetch_granularity); returns the
    previous value."""
    prev = C.c_int32(0)
    _check(load().tango_set_l2_fetch_granularity(int(nbytes), C.byref(prev)), "tango_set_l2_fetch_granularity")
    return int(prev.value)


def launch_count() -> int:
    return int(load().tango_launch_count())


def profile_read(reset: bool = True) -> dict:
    """{kernel name: (total device ms, launches)} since the last reset (waits for pending events)."""
    L = load()
    _check(L.tango_profile_collect(), "tango_profile_collect")
    out = {}
    buf = C.create_string_buffer(64)
    ms, cnt = C.c_double(), C.c_int64()
    for i in range(L.tango_profile_num_entries()):
        _check(L.tango_profile_entry(i, buf, 64, C.byref(ms), C.byref(cnt)), "tango_profile_entry")
        if cnt.value:
            out[buf.value.decode()] = (ms.value, cnt.value)
    if reset:
        L.tango_profile_reset()
    return out


# ---------------------------------------------------------------------------------------- graph
class DeviceGraph:
    """A graph (paper_2308_00890_b200.inputs.Graph) resident on the GPU, viewed as a tango_graph.

    With row_begin/row_end the view covers this rank's node block (destination-row partitioning);
    the in/out CSR arrays are then sliced to the owned rows.
    """

    _next_id = 0

    def __init__(self, g, device="cuda", chunk=256, row_begin=0, row_end=None, keep_eid=None):
        lg = local_graph(g, row_begin, row_end, keep_eid)
        t = lambda a: torch.from_numpy(a).to(device)
        self.in_ptr, self.in_src = t(lg.in_ptr), t(lg.in_src)
        self.out_ptr, self.out_dst = t(lg.out_ptr), t(lg.out_dst)
        self.out_eid = t(lg.out_eid) if lg.out_eid is not None else None
        self.n_global, self.row_begin, self.row_end = g.n, lg.row_begin, lg.row_end
        self.n_local = lg.n
        self.e_in, self.e_out = lg.e, lg.e_out
        self.chunk = chunk
        DeviceGraph._next_id += 1   # a process-unique id per device graph: the layers' static-plan cache key
        self.struct = Graph(g.n, lg.row_begin, lg.row_end, _ptr(self.in_ptr), _ptr(self.in_src) if self.e_in else None,
                            self.e_in, _ptr(self.out_ptr), _ptr(self.out_dst) if self.e_out else None,
                            _ptr(self.out_eid) if self.out_eid is not None and self.e_out else None, self.e_out,
                            chunk, DeviceGraph._next_id)

    def ref(self):
        return C.byref(self.struct)


def qtensor(q, scale, rows, cols, bits=8):
    return QTensor(_ptr(q), _ptr(scale), rows, cols, q.shape[1] if q.dim() == 2 else cols, bits)


# ---------------------------------------------------------------------------------------- primitives
def quantize(x, bits=8, seed=0, step=0, tag=0, global_row0=0, amax_hint=None, ld=None, status=None, want_amax=True):
    """tango_quantize: returns (q int8 [rows, ld], scale f32 (1,), amax f32 (1,) or None)."""
    L = load()
    x = x.contiguous()
    rows, cols = x.shape
    ld = ld if ld is not None else ld32(cols)
    q = torch.empty((rows, ld), dtype=torch.int8, device=x.device)
    s = torch.empty(1, dtype=torch.float32, device=x.device)
    amax = torch.empty(1, dtype=torch.float32, device=x.device) if want_amax else None
    qt = QTensor(_ptr(q), _ptr(s), rows, cols, ld, bits)
    _check(L.tango_quantize(_ptr(x), rows, cols, global_row0, _ptr(amax_hint), Rng(seed, step, tag), C.byref(qt),
                            _ptr(amax), _ptr(status), _stream()), "tango_quantize")
    return q, s, amax


def gemm_q(A, sA, a_layout, B, sB, b_layout, M, N, K, want=("f32",), bits=8):
    """tango_gemm_q. A/B: int8 2-D tensors (stored layouts per a_layout/b_layout)."""
    L = load()
    arows, acols = (K, M) if a_layout == TANGO_MN_MAJOR else (M, K)
    brows, bcols = (K, N) if b_layout == TANGO_MN_MAJOR else (N, K)
    qa = QTensor(_ptr(A), _ptr(sA), arows, acols, A.shape[1], bits)
    qb = QTensor(_ptr(B), _ptr(sB), brows, bcols, B.shape[1], bits)
    dev = A.device
    out = {}
    Cf = torch.empty((M, N), dtype=torch.float32, device=dev) if "f32" in want else None
    Ci = torch.empty((M, N), dtype=torch.int32, device=dev) if "i32" in want else None
    Cl = torch.empty((M, N), dtype=torch.int64, device=dev) if "i64" in want else None
    _check(L.tango_gemm_q(C.byref(qa), a_layout, C.byref(qb), b_layout, M, N, K, _ptr(Cf), _ptr(Ci), _ptr(Cl),
                          _stream()), "tango_gemm_q")
    if Cf is not None:
        out["f32"] = Cf
    if Ci is not None:
        out["i32"] = Ci
    if Cl is not None:
        out["i64"] = Cl
    return out


def sddmm_add(graph: DeviceGraph, qS, sS, qD, sD, heads, slope):
    L = load()
    e_pre = torch.empty((graph.e_in, heads), dtype=torch.float32, device="cuda")
    el = torch.empty_like(e_pre)
    xs = QTensor(_ptr(qS), _ptr(sS), qS.shape[0], heads, heads, 8)
    xd = QTensor(_ptr(qD), _ptr(sD), qD.shape[0], heads, heads, 8)
    _check(L.tango_sddmm_q(graph.ref(), TANGO_SDDMM_ADD, C.byref(xs), C.byref(xd), heads, slope, _ptr(e_pre),
                           _ptr(el), None, _stream()), "tango_sddmm_q(add)")
    return e_pre, el


def sddmm_dot(graph: DeviceGraph, qA_dst, sA, qB_src, sB, heads, cols):
    L = load()
    out = torch.empty((graph.e_in, heads), dtype=torch.float32, device="cuda")
    acc = torch.empty((graph.e_in, heads), dtype=torch.int32, device="cuda")
    xs = QTensor(_ptr(qB_src), _ptr(sB), qB_src.shape[0], cols, qB_src.shape[1], 8)
    xd = QTensor(_ptr(qA_dst), _ptr(sA), qA_dst.shape[0], cols, qA_dst.shape[1], 8)
    _check(L.tango_sddmm_q(graph.ref(), TANGO_SDDMM_DOT, C.byref(xs), C.byref(xd), heads, 0.0, _ptr(out), None,
                           _ptr(acc), _stream()), "tango_sddmm_q(dot)")
    return out, acc


def edge_softmax(graph: DeviceGraph, heads, el):
    L = load()
    m = torch.empty((graph.n_global, heads), dtype=torch.float32, device="cuda")
    den = torch.empty_like(m)
    alpha = torch.empty((graph.e_in, heads), dtype=torch.float32, device="cuda")
    _check(L.tango_edge_softmax(graph.ref(), heads, _ptr(el.contiguous()), _ptr(m), _ptr(den), _ptr(alpha),
                                _stream()), "tango_edge_softmax")
    return m, den, alpha


def softmax_bwd(graph: DeviceGraph, heads, alpha, dalpha, e_pre, slope):
    L = load()
    P = torch.empty((graph.n_global, heads), dtype=torch.float32, device="cuda")
    dEp = torch.empty((graph.e_in, heads), dtype=torch.float32, device="cuda")
    _check(L.tango_softmax_bwd(graph.ref(), heads, _ptr(alpha), _ptr(dalpha), _ptr(e_pre), slope, _ptr(P),
                               _ptr(dEp), _stream()), "tango_softmax_bwd")
    return P, dEp


def spmm(graph: DeviceGraph, direction, qX, sX, cols, heads, edge_w=None, row_scale=None, amax_out=None,
         out=None):
    """tango_spmm_q: weighted (edge_w [E][heads] fp32, Σᶜ fmaf) or unweighted (exact int32) aggregation of
    int8 rows; optional per-row scale and amax(|out|) (amax_out is raised, not reset)."""
    L = load()
    x = QTensor(_ptr(qX), _ptr(sX), qX.shape[0], cols, qX.shape[1], 8)
    out = out if out is not None else torch.empty((graph.n_local, cols), dtype=torch.float32, device="cuda")
    oi = None if edge_w is not None else torch.empty((graph.n_local, cols), dtype=torch.int32, device="cuda")
    _check(L.tango_spmm_q(graph.ref(), direction, _ptr(edge_w), C.byref(x), heads, _ptr(row_scale), _ptr(out),
                          _ptr(oi), _ptr(amax_out), _stream()), "tango_spmm_q")
    return out, oi


def spmm_q8(graph: DeviceGraph, direction, qa, sa, qX, sX, cols, heads, out=None, out_i32=None, want_f32=True):
    """tango_spmm_q8 (NEXT-4 int8-α SPMM): qa int8 [e_in, heads] edge codes (in-CSR slot order) with scale sa,
    qX int8 [N, ld] node codes; returns (out f32 or None, out_i32)."""
    L = load()
    a = QTensor(_ptr(qa), _ptr(sa), qa.shape[0], heads, heads, 8)
    x = QTensor(_ptr(qX), _ptr(sX), qX.shape[0], cols, qX.shape[1], 8)
    out_i32 = out_i32 if out_i32 is not None else torch.empty((graph.n_local, cols), dtype=torch.int32, device="cuda")
    if want_f32 and out is None:
        out = torch.empty((graph.n_local, cols), dtype=torch.float32, device="cuda")
    _check(L.tango_spmm_q8(graph.ref(), direction, C.byref(a), C.byref(x), heads, _ptr(out_i32),
                           _ptr(out) if want_f32 else None, _stream()), "tango_spmm_q8")
    return (out if want_f32 else None), out_i32


def edge_sum(graph: DeviceGraph, direction, heads, x, out=None):
    L = load()
    out = out if out is not None else torch.empty((graph.n_local, heads), dtype=torch.float32, device="cuda")
    _check(L.tango_edge_sum(graph.ref(), direction, heads, _ptr(x.contiguous()), _ptr(out), _stream()),
           "tango_edge_sum")
    return out


# ---------------------------------------------------------------------------------------- layers
class Comm:
    """NCCL communicator (tango_comm) for destination-row partitioning; the unique id is
    broadcast by the caller (torch.distributed)."""

    def __init__(self, nranks, rank, unique_id: bytes, row_starts, always=False, reserve_row_bytes=0):
        L = load()
        self.handle = C.c_void_p()
        buf = C.create_string_buffer(unique_id, len(unique_id))
        _check(L.tango_comm_init(C.byref(self.handle), buf, nranks, rank), "tango_comm_init")
        starts = np.ascontiguousarray(row_starts, dtype=np.int64)
        _check(L.tango_comm_set_partition(self.handle, starts.ctypes.data), "tango_comm_set_partition")
        if always:
            _check(L.tango_comm_set_options(self.handle, 1), "tango_comm_set_options")
        if reserve_row_bytes:
            self.reserve(reserve_row_bytes)

    def reserve(self, max_row_bytes: int):
        """Staging of the padded ncclAllGather for node rows of up to max_row_bytes bytes."""
        _check(load().tango_comm_reserve(self.handle, int(max_row_bytes)), "tango_comm_reserve")

    def nccl_calls(self) -> int:
        return int(load().tango_comm_nccl_calls(self.handle))

    @classmethod
    def local(cls, group: "LocalGroup", rank, row_starts):
        """Loopback communicator of an in-process group (one host thread per rank, one GPU)."""
        L = load()
        self = cls.__new__(cls)
        self.handle = C.c_void_p()
        _check(L.tango_comm_init_local(C.byref(self.handle), group.handle, rank), "tango_comm_init_local")
        starts = np.ascontiguousarray(row_starts, dtype=np.int64)
        _check(L.tango_comm_set_partition(self.handle, starts.ctypes.data), "tango_comm_set_partition")
        return self

    @staticmethod
    def unique_id() -> bytes:
        L = load()
        n = L.tango_comm_unique_id_bytes()
        buf = C.create_string_buffer(n)
        _check(L.tango_comm_get_unique_id(buf), "tango_comm_get_unique_id")
        return buf.raw

    def close(self):
        if self.handle:
            load().tango_comm_destroy(self.handle)
            self.handle = C.c_void_p()


def quant_error(x, q, s, bits=8):
    """tango_quant_error: Error_X (Eq.4) of codes q [rows, ld] with scale s (1,) against x [rows, cols]."""
    L = load()
    x = x.contiguous()
    rows, cols = x.shape
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    qt = QTensor(_ptr(q), _ptr(s), rows, cols, q.shape[1], bits)
    _check(L.tango_quant_error(_ptr(x), rows, cols, C.byref(qt), _ptr(out), _stream()), "tango_quant_error")
    return out


def select_bits(x, threshold=0.3, bmin=2, bmax=8):
    """tango_select_bits: (bits int32 (1,), errs float64 (bmax-bmin+1,)); bits < 0: none qualified."""
    L = load()
    x = x.contiguous()
    errs = torch.empty(bmax - bmin + 1, dtype=torch.float64, device=x.device)
    bits = torch.empty(1, dtype=torch.int32, device=x.device)
    _check(L.tango_select_bits(_ptr(x), x.numel(), threshold, bmin, bmax, _ptr(errs), _ptr(bits), _stream()),
           "tango_select_bits")
    return bits, errs


class LocalGroup:
    """tango_local_group: nranks in-process ranks exchanging through device memory (tests)."""

    def __init__(self, nranks):
        L = load()
        self.handle = C.c_void_p()
        _check(L.tango_local_group_create(C.byref(self.handle), nranks), "tango_local_group_create")

    def close(self):
        if self.handle:
            load().tango_local_group_destroy(self.handle)
            self.handle = C.c_void_p()


class GATLayer:
    """One quantized GAT layer (tango_gat_layer_fwd / _bwd) with its device ctx."""

    def __init__(self, graph: DeviceGraph, W, a_src, a_dst, heads, head_dim, slope=0.2, bits=8, comm: Comm = None):
        L = load()
        self.graph, self.heads, self.head_dim, self.bits = graph, heads, head_dim, bits
        self.W, self.a_src, self.a_dst = W.contiguous(), a_src.contiguous(), a_dst.contiguous()
        self.F = W.shape[0]
        self.HD = heads * head_dim
        self.params = GatParams(_ptr(self.W), _ptr(self.a_src), _ptr(self.a_dst), self.F, heads, head_dim, slope, bits)
        nbytes = L.tango_gat_ctx_bytes(graph.ref(), C.byref(self.params))
        if nbytes == 0:
            raise TangoError(2, "tango_gat_ctx_bytes")
        self.ctx = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.comm = comm

    def _comm(self):
        return self.comm.handle if self.comm is not None else None

    def forward(self, H, seed=0x7A4E60, step=0, layer_id=0, amax_hint=None, out=None, amax_out=None):
        L = load()
        n = self.graph.n_local
        out = out if out is not None else torch.empty((n, self.HD), dtype=torch.float32, device="cuda")
        amax_out = amax_out if amax_out is not None else torch.empty(1, dtype=torch.float32, device="cuda")
        _check(L.tango_gat_layer_fwd(self.graph.ref(), C.byref(self.params), _arg(H, "H", (n, self.F)),
                                     _arg(amax_hint, "amax_hint", (1,), optional=True), Rng(seed, step, 0), layer_id,
                                     _ptr(self.ctx), self.ctx.numel(), _arg(out, "out", (n, self.HD)),
                                     _arg(amax_out, "amax_out", (1,)), self._comm(), _ptr(self.status), _stream()),
               "tango_gat_layer_fwd")
        return out, amax_out

    def backward(self, dH_out, seed=0x7A4E60, step=0, layer_id=0, amax_hint=None, want_dH=True, outs=None):
        L = load()
        n = self.graph.n_local
        if outs is None:
            dH = torch.empty((n, self.F), dtype=torch.float32, device="cuda") if want_dH else None
            dW = torch.empty((self.F, self.HD), dtype=torch.float32, device="cuda")
            da_s = torch.empty(self.HD, dtype=torch.float32, device="cuda")
            da_d = torch.empty(self.HD, dtype=torch.float32, device="cuda")
        else:
            dH, dW, da_s, da_d = outs
        _check(L.tango_gat_layer_bwd(self.graph.ref(), C.byref(self.params), _ptr(self.ctx), self.ctx.numel(),
                                     _arg(dH_out, "dH_out", (n, self.HD)),
                                     _arg(amax_hint, "amax_hint", (1,), optional=True), Rng(seed, step, 0), layer_id,
                                     _arg(dH, "dH", (n, self.F), optional=True), _arg(dW, "dW", (self.F, self.HD)),
                                     _arg(da_s, "da_src", (self.HD,)), _arg(da_d, "da_dst", (self.HD,)), None,
                                     self._comm(), _ptr(self.status), _stream()),
               "tango_gat_layer_bwd")
        return dH, dW, da_s, da_d

    def view_dataflow(self) -> int:
        """1: round-1 kernels (gat.cu), 2: v6 single-GPU dataflow (gat2.cu)."""
        v = GatCtxView()
        _check(load().tango_gat_ctx_get_view(self.graph.ref(), C.byref(self.params), _ptr(self.ctx), C.byref(v)),
               "tango_gat_ctx_get_view")
        return int(v.dataflow)

    def view(self):
        """Device tensors inside ctx (copies), for parity tests."""
        L = load()
        v = GatCtxView()
        _check(L.tango_gat_ctx_get_view(self.graph.ref(), C.byref(self.params), _ptr(self.ctx), C.byref(v)),
               "tango_gat_ctx_get_view")
        base = self.ctx.data_ptr()
        N, n, H, HD, F, E = self.graph.n_global, self.graph.n_local, self.heads, self.HD, self.F, self.graph.e_in

        def sl(p, nbytes, dtype, shape):
            off = p - base
            return self.ctx[off:off + nbytes].view(dtype).reshape(shape).clone()

        i8, f4 = torch.int8, torch.float32
        out = dict(
            qH=sl(v.qH, n * v.ldF, i8, (n, v.ldF))[:, :F], qW=sl(v.qW, F * v.ldHD, i8, (F, v.ldHD))[:, :HD],
            qWt=sl(v.qWt, HD * v.ldFt, i8, (HD, v.ldFt))[:, :F],
            qHp=sl(v.qHp, N * v.ldHD, i8, (N, v.ldHD))[:, :HD], qS=sl(v.qS, N * H, i8, (N, H)),
            qD=sl(v.qD, N * H, i8, (N, H)), qG=sl(v.qG, N * v.ldHD, i8, (N, v.ldHD))[:, :HD],
            qdHp=sl(v.qdHp, n * v.ldHD, i8, (n, v.ldHD))[:, :HD],
            qH_full=sl(v.qH, n * v.ldF, i8, (n, v.ldF)), qHp_full=sl(v.qHp, N * v.ldHD, i8, (N, v.ldHD)),
            S=sl(v.S, n * H * 4, f4, (n, H)), D=sl(v.D, n * H * 4, f4, (n, H)), m=sl(v.m, N * H * 4, f4, (N, H)),
            den=sl(v.den, N * H * 4, f4, (N, H)), P=sl(v.P, N * H * 4, f4, (N, H)),
            dD=sl(v.dD, N * H * 4, f4, (N, H)), dHp=sl(v.dHp, n * HD * 4, f4, (n, HD)),
            dalpha=sl(v.dalpha, E * H * 4, f4, (E, H)), scalars=sl(v.scalars, 64 * 4, f4, (64,)))
        if v.codes_biased:   # excess-128 storage of q_H′ / q_G -> plain codes
            flip = torch.tensor(-128, dtype=i8, device=self.ctx.device)
            out["qHp"] = torch.bitwise_xor(out["qHp"], flip)
            out["qG"] = torch.bitwise_xor(out["qG"], flip)
        out["codes_biased"] = bool(v.codes_biased)
        out["dS"] = sl(v.dS, N * H * 4, f4, (N, H))
        out["dataflow"] = int(v.dataflow)
        if v.dataflow == 1:
            pack = sl(v.alpha_pack, E * 2 * H * 4, f4, (E, 2 * H))
            out["alpha"] = pack[:, :H].abs()
            out["e_pre_pos"] = ~torch.signbit(pack[:, :H])
            out["dE_pre"] = pack[:, H:]
        else:
            out["dalpha_out"] = sl(v.alpha_pack, self.graph.e_out * H * 4, f4, (self.graph.e_out, H))
        return out

    def check_status(self):
        st = int(self.status.item())
        if st != 0:
            raise TangoError(st, "device status")


class GCNLayer:
    """One quantized GCN layer (tango_gcn_layer_fwd / _bwd)."""

    def __init__(self, graph: DeviceGraph, W, bits=8, comm: Comm = None):
        L = load()
        self.graph, self.bits = graph, bits
        self.W = W.contiguous()
        self.F, self.O = W.shape
        self.params = GcnParams(_ptr(self.W), self.F, self.O, bits)
        nbytes = L.tango_gcn_ctx_bytes(graph.ref(), C.byref(self.params))
        if nbytes == 0:
            raise TangoError(2, "tango_gcn_ctx_bytes")
        self.ctx = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.comm = comm

    def forward(self, X, seed=0x7A4E60, step=0, layer_id=0, amax_hint=None, out=None, amax_out=None):
        L = load()
        out = out if out is not None else torch.empty((self.graph.n_local, self.O), dtype=torch.float32,
                                                      device="cuda")
        amax_out = amax_out if amax_out is not None else torch.empty(1, dtype=torch.float32, device="cuda")
        n = self.graph.n_local
        _check(L.tango_gcn_layer_fwd(self.graph.ref(), C.byref(self.params), _arg(X, "X", (n, self.F)),
                                     _arg(amax_hint, "amax_hint", (1,), optional=True), Rng(seed, step, 0), layer_id,
                                     _ptr(self.ctx), self.ctx.numel(), _arg(out, "out", (n, self.O)),
                                     _arg(amax_out, "amax_out", (1,)), self.comm.handle if self.comm else None,
                                     _ptr(self.status), _stream()), "tango_gcn_layer_fwd")
        return out, amax_out

    def backward(self, dout, seed=0x7A4E60, step=0, layer_id=0, want_dX=True, outs=None):
        L = load()
        if outs is None:
            dX = torch.empty((self.graph.n_local, self.F), dtype=torch.float32, device="cuda") if want_dX else None
            dW = torch.empty((self.F, self.O), dtype=torch.float32, device="cuda")
        else:
            dX, dW = outs
        n = self.graph.n_local
        _check(L.tango_gcn_layer_bwd(self.graph.ref(), C.byref(self.params), _ptr(self.ctx), self.ctx.numel(),
                                     _arg(dout, "dout", (n, self.O)), Rng(seed, step, 0), layer_id,
                                     _arg(dX, "dX", (n, self.F), optional=True), _arg(dW, "dW", (self.F, self.O)),
                                     self.comm.handle if self.comm else None, _ptr(self.status), _stream()),
               "tango_gcn_layer_bwd")
        return dX, dW

    def check_status(self):
        st = int(self.status.item())
        if st != 0:
            raise TangoError(st, "device status")

    def view(self):
        L = load()
        v = GcnCtxView()
        _check(L.tango_gcn_ctx_get_view(self.graph.ref(), C.byref(self.params), _ptr(self.ctx), C.byref(v)),
               "tango_gcn_ctx_get_view")
        base = self.ctx.data_ptr()
        N, n, F, O = self.graph.n_global, self.graph.n_local, self.F, self.O

        def sl(p, nbytes, dtype, shape):
            off = p - base
            return self.ctx[off:off + nbytes].view(dtype).reshape(shape).clone()

        i8 = torch.int8
        return dict(qX=sl(v.qX, n * v.ldF, i8, (n, v.ldF))[:, :F], qW=sl(v.qW, F * v.ldO, i8, (F, v.ldO))[:, :O],
                    qYs=sl(v.qYs, N * v.ldO, i8, (N, v.ldO))[:, :O], qGs=sl(v.qGs, N * v.ldO, i8, (N, v.ldO))[:, :O],
                    qdY=sl(v.qdY, n * v.ldO, i8, (n, v.ldO))[:, :O], ia=sl(v.ia, n * O * 4, torch.int32, (n, O)),
                    ib=sl(v.ib, n * O * 4, torch.int32, (n, O)),
                    scalars=sl(v.scalars, 64 * 4, torch.float32, (64,)))


# ---------------------------------------------------------------------------------------- NEXT-1
def sgemm(A, B, a_layout=TANGO_K_MAJOR, b_layout=TANGO_MN_MAJOR, out=None, workspace=None):
    """tango_sgemm (full-precision GEMM, reading R33).  Default layouts: A [M][K], B [K][N]."""
    L = load()
    M, K = (A.shape[1], A.shape[0]) if a_layout == TANGO_MN_MAJOR else A.shape
    N = B.shape[0] if b_layout == TANGO_K_MAJOR else B.shape[1]
    out = out if out is not None else torch.empty((M, N), dtype=torch.float32, device=A.device)
    need = L.tango_sgemm_workspace_bytes(M, N, K)
    if workspace is None and need:
        workspace = torch.empty(need, dtype=torch.uint8, device=A.device)
    _check(L.tango_sgemm(_ptr(A), A.shape[1], a_layout, _ptr(B), B.shape[1], b_layout, M, N, K, _ptr(out),
                         _ptr(workspace), workspace.numel() if workspace is not None else 0, _stream()),
           "tango_sgemm")
    return out


def colsum(x, out=None, workspace=None):
    L = load()
    rows, cols = x.shape
    out = out if out is not None else torch.empty(cols, dtype=torch.float32, device=x.device)
    need = L.tango_colsum_workspace_bytes(rows, cols)
    if workspace is None and need:
        workspace = torch.empty(need, dtype=torch.uint8, device=x.device)
    _check(L.tango_colsum(_ptr(x), rows, cols, _ptr(out), _ptr(workspace),
                          workspace.numel() if workspace is not None else 0, _stream()), "tango_colsum")
    return out


def bias_act_fwd(x, bias, out=None, amax_out=None):
    """tango_bias_act_fwd: (ReLU(x + b), max of it)."""
    L = load()
    rows, cols = x.shape
    out = out if out is not None else torch.empty_like(x)
    amax_out = amax_out if amax_out is not None else torch.empty(1, dtype=torch.float32, device=x.device)
    _check(L.tango_bias_act_fwd(_ptr(x), _ptr(bias), rows, cols, _ptr(out), _ptr(amax_out), _stream()),
           "tango_bias_act_fwd")
    return out, amax_out


def bias_act_bwd(y, dy, dx=None, dbias=None, amax_out=None, workspace=None):
    """tango_bias_act_bwd: (dx, dbias, max|dx|)."""
    L = load()
    rows, cols = y.shape
    dx = dx if dx is not None else torch.empty_like(y)
    dbias = dbias if dbias is not None else torch.empty(cols, dtype=torch.float32, device=y.device)
    amax_out = amax_out if amax_out is not None else torch.empty(1, dtype=torch.float32, device=y.device)
    need = L.tango_colsum_workspace_bytes(rows, cols)
    if workspace is None and need:
        workspace = torch.empty(need, dtype=torch.uint8, device=y.device)
    _check(L.tango_bias_act_bwd(_ptr(y), _ptr(dy), rows, cols, _ptr(dx), _ptr(dbias), _ptr(amax_out),
                                _ptr(workspace), workspace.numel() if workspace is not None else 0, _stream()),
           "tango_bias_act_bwd")
    return dx, dbias, amax_out


def cross_entropy(logits, labels, n_labeled, dlogits=None, loss=None, status=None):
    """tango_cross_entropy: (loss f64 (1,), dlogits)."""
    L = load()
    rows, classes = logits.shape
    dlogits = dlogits if dlogits is not None else torch.empty_like(logits)
    loss = loss if loss is not None else torch.empty(1, dtype=torch.float64, device=logits.device)
    _check(L.tango_cross_entropy(_ptr(logits), _ptr(labels), rows, classes, int(n_labeled), _ptr(dlogits),
                                 _ptr(loss), _ptr(status), _stream()), "tango_cross_entropy")
    return loss, dlogits


def sgd_update(pairs, lr):
    """tango_sgd_update over [(w, g), ...] (in place on w)."""
    L = load()
    arr = (SgdTensor * len(pairs))(*[SgdTensor(_ptr(w), _ptr(g), w.numel()) for w, g in pairs])
    _check(L.tango_sgd_update(arr, len(pairs), float(lr), _stream()), "tango_sgd_update")


class GATOutLayer:
    """The full-precision final GAT layer (tango_gat_out_fwd / _bwd) with its device ctx."""

    def __init__(self, graph: DeviceGraph, W, a_src, a_dst, bias, heads, classes, slope=0.2):
        L = load()
        self.graph, self.heads, self.classes = graph, heads, classes
        self.W, self.a_src, self.a_dst, self.bias = (t.contiguous() for t in (W, a_src, a_dst, bias))
        self.F = W.shape[0]
        self.HC = heads * classes
        self.params = GatOutParams(_ptr(self.W), _ptr(self.a_src), _ptr(self.a_dst), _ptr(self.bias), self.F, heads,
                                   classes, slope)
        nbytes = L.tango_gat_out_ctx_bytes(graph.ref(), C.byref(self.params))
        if nbytes == 0:
            raise TangoError(2, "tango_gat_out_ctx_bytes")
        self.ctx = torch.empty(nbytes, dtype=torch.uint8, device="cuda")

    def forward(self, H, out=None):
        L = load()
        out = out if out is not None else torch.empty((self.graph.n_local, self.classes), dtype=torch.float32,
                                                      device="cuda")
        _check(L.tango_gat_out_fwd(self.graph.ref(), C.byref(self.params), _ptr(H), _ptr(self.ctx), self.ctx.numel(),
                                   _ptr(out), _stream()), "tango_gat_out_fwd")
        return out

    def backward(self, H, dlogits, want_dH=True, outs=None):
        L = load()
        n = self.graph.n_local
        if outs is None:
            dH = torch.empty((n, self.F), dtype=torch.float32, device="cuda") if want_dH else None
            dW = torch.empty((self.F, self.HC), dtype=torch.float32, device="cuda")
            da_s = torch.empty(self.HC, dtype=torch.float32, device="cuda")
            da_d = torch.empty(self.HC, dtype=torch.float32, device="cuda")
            db = torch.empty(self.classes, dtype=torch.float32, device="cuda")
        else:
            dH, dW, da_s, da_d, db = outs
        _check(L.tango_gat_out_bwd(self.graph.ref(), C.byref(self.params), _ptr(self.ctx), self.ctx.numel(), _ptr(H),
                                   _ptr(dlogits), _ptr(dH), _ptr(dW), _ptr(da_s), _ptr(da_d), _ptr(db), _stream()),
               "tango_gat_out_bwd")
        return dH, dW, da_s, da_d, db

    def view(self):
        L = load()
        v = GatOutCtxView()
        _check(L.tango_gat_out_ctx_get_view(self.graph.ref(), C.byref(self.params), _ptr(self.ctx), C.byref(v)),
               "tango_gat_out_ctx_get_view")
        base = self.ctx.data_ptr()
        n, H, E, HC, Cc = self.graph.n_local, self.heads, self.graph.e_in, self.HC, self.classes
        shapes = dict(Hp=(n, HC), S=(n, H), D=(n, H), e_pre=(E, H), alpha=(E, H), m=(n, H), den=(n, H), G=(n, Cc),
                      dalpha=(E, H), dE_pre=(E, H), P=(n, H), dD=(n, H), dS=(n, H), dHp=(n, HC), agg=(n, HC))
        out = {}
        for f, shp in shapes.items():
            off = getattr(v, f) - base
            cnt = shp[0] * shp[1]
            out[f] = self.ctx[off:off + 4 * cnt].view(torch.float32).reshape(shp).clone()
        return out


class GCNOutLayer:
    """The full-precision final GCN layer (tango_gcn_out_fwd / _bwd) with its device ctx."""

    def __init__(self, graph: DeviceGraph, W, bias):
        L = load()
        self.graph = graph
        self.W, self.bias = W.contiguous(), bias.contiguous()
        self.F, self.classes = W.shape
        self.params = GcnOutParams(_ptr(self.W), _ptr(self.bias), self.F, self.classes)
        nbytes = L.tango_gcn_out_ctx_bytes(graph.ref(), C.byref(self.params))
        if nbytes == 0:
            raise TangoError(2, "tango_gcn_out_ctx_bytes")
        self.ctx = torch.empty(nbytes, dtype=torch.uint8, device="cuda")

    def forward(self, X, out=None):
        out = out if out is not None else torch.empty((self.graph.n_local, self.classes), dtype=torch.float32,
                                                      device="cuda")
        _check(load().tango_gcn_out_fwd(self.graph.ref(), C.byref(self.params), _ptr(X), _ptr(self.ctx),
                                        self.ctx.numel(), _ptr(out), _stream()), "tango_gcn_out_fwd")
        return out

    def backward(self, X, dlogits, want_dX=True, outs=None):
        n = self.graph.n_local
        if outs is None:
            dX = torch.empty((n, self.F), dtype=torch.float32, device="cuda") if want_dX else None
            dW = torch.empty((self.F, self.classes), dtype=torch.float32, device="cuda")
            db = torch.empty(self.classes, dtype=torch.float32, device="cuda")
        else:
            dX, dW, db = outs
        _check(load().tango_gcn_out_bwd(self.graph.ref(), C.byref(self.params), _ptr(self.ctx), self.ctx.numel(),
                                        _ptr(X), _ptr(dlogits), _ptr(dX), _ptr(dW), _ptr(db), _stream()),
               "tango_gcn_out_bwd")
        return dX, dW, db

    def view(self):
        v = GcnOutCtxView()
        _check(load().tango_gcn_out_ctx_get_view(self.graph.ref(), C.byref(self.params), _ptr(self.ctx), C.byref(v)),
               "tango_gcn_out_ctx_get_view")
        base, n, Cc = self.ctx.data_ptr(), self.graph.n_local, self.classes
        out = {}
        for f in ("Y", "Ys", "agg", "Gs", "aggb", "dY"):
            off = getattr(v, f) - base
            out[f] = self.ctx[off:off + 4 * n * Cc].view(torch.float32).reshape(n, Cc).clone()
        return out


# ---------------------------------------------------------------------------------------- NEXT-4
def quantize_int4(x, seed=0, step=0, tag=0, global_row0=0, amax_hint=None, ld_bytes=None, status=None):
    """tango_quantize_int4: (packed uint8 [rows, ld_bytes], scale (1,), amax (1,))."""
    x = x.contiguous()
    rows, cols = x.shape
    ld_bytes = ld_bytes if ld_bytes is not None else (cols // 2 + 3) // 4 * 4
    q = torch.zeros((rows, ld_bytes), dtype=torch.uint8, device=x.device)
    s = torch.empty(1, dtype=torch.float32, device=x.device)
    amax = torch.empty(1, dtype=torch.float32, device=x.device)
    _check(load().tango_quantize_int4(_ptr(x), rows, cols, global_row0, _ptr(amax_hint), Rng(seed, step, tag), _ptr(q),
                                      ld_bytes, _ptr(s), _ptr(amax), _ptr(status), _stream()), "tango_quantize_int4")
    return q, s, amax


def sddmm_qn(graph: DeviceGraph, op, bits, Xsrc, s_src, Xdst, s_dst, heads, cols, slope=0.2, out0=None, out1=None):
    """tango_sddmm_qn on int8 (bits 8) or packed int4 (bits 4) rows; returns (out0, out1)."""
    E = graph.e_in
    out0 = out0 if out0 is not None else torch.empty((E, heads), dtype=torch.float32, device="cuda")
    if op == TANGO_SDDMM_ADD and out1 is None:
        out1 = torch.empty((E, heads), dtype=torch.float32, device="cuda")
    _check(load().tango_sddmm_qn(graph.ref(), op, bits, _ptr(Xsrc), Xsrc.shape[1] * Xsrc.element_size(), _ptr(s_src),
                                 _ptr(Xdst), Xdst.shape[1] * Xdst.element_size(), _ptr(s_dst), heads, cols, slope,
                                 _ptr(out0), _ptr(out1), _stream()), "tango_sddmm_qn")
    return out0, out1
