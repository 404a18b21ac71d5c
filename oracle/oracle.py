"""ctypes binding of the CPU oracle (oracle/tango_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module.  The product path
(paper_2308_00890_b200) never imports it.

``build()`` compiles liboracle.so with gcc (-O2 -ffp-contract=off
-fno-fast-math -fopenmp) next to the C source.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tango_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fno-finite-math-only",
          "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wno-unknown-pragmas"]

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Graph(C.Structure):
    _fields_ = [("n", C.c_int64), ("e", C.c_int64), ("in_ptr", C.c_void_p), ("in_src", C.c_void_p),
                ("chunk", C.c_int32)]


class QRef(C.Structure):
    _fields_ = [("q", C.c_void_p), ("v", C.c_void_p), ("s", C.c_float)]


class Cfg(C.Structure):
    _fields_ = [("F", C.c_int32), ("H", C.c_int32), ("D", C.c_int32), ("slope", C.c_float),
                ("bits", C.c_int32), ("seed", C.c_uint64), ("step", C.c_uint32), ("layer_id", C.c_uint32)]


_P = C.c_void_p
_FWD_FIELDS = ["qH", "sH", "qW", "sW", "maxacc", "Hp", "S", "Dd", "qHp", "sHp", "qS", "sS", "qD", "sD",
               "e_pre", "alpha", "m", "den", "Hout", "amax_out"]
_BWD_FIELDS = ["qG", "sG", "dalpha", "P", "dE", "dE_pre", "dD", "dS", "dHp_agg", "dHp", "da_src", "da_dst",
               "da_src_abs", "da_dst_abs", "qdHp", "sdHp", "dH", "dW"]
_GCN_FWD_FIELDS = ["qX", "sX", "qW", "sW", "Ys", "qYs", "sYs", "ia", "out"]
_GCN_BWD_FIELDS = ["Gs", "qGs", "sGs", "ib", "dY", "qdY", "sdY", "dX", "dW"]


class FwdOut(C.Structure):
    _fields_ = [(f, _P) for f in _FWD_FIELDS]


class BwdOut(C.Structure):
    _fields_ = [(f, _P) for f in _BWD_FIELDS]


class GcnFwdOut(C.Structure):
    _fields_ = [(f, _P) for f in _GCN_FWD_FIELDS]


class GcnBwdOut(C.Structure):
    _fields_ = [(f, _P) for f in _GCN_BWD_FIELDS]


class OutCfg(C.Structure):
    _fields_ = [("F", C.c_int32), ("H", C.c_int32), ("C", C.c_int32), ("slope", C.c_float)]


_OUT_FWD_FIELDS = ["Hp", "S", "Dd", "e_pre", "alpha", "m", "den", "agg", "logits"]
_OUT_BWD_FIELDS = ["db", "G", "dalpha", "P", "dE", "dE_pre", "dD", "dS", "dHp_agg", "dHp", "da_src", "da_dst",
                   "da_src_abs", "da_dst_abs", "dH", "dW"]


class GcnOutFwdOut(C.Structure):
    _fields_ = [(f, _P) for f in ("Y", "Ys", "agg", "logits")]


class GcnOutBwdOut(C.Structure):
    _fields_ = [(f, _P) for f in ("db", "Gs", "aggb", "dY", "dX", "dW")]


class OutFwdOut(C.Structure):
    _fields_ = [(f, _P) for f in _OUT_FWD_FIELDS]


class OutBwdOut(C.Structure):
    _fields_ = [(f, _P) for f in _OUT_BWD_FIELDS]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_philox4x32_10.argtypes = [_P, _P, _P]
        L.orc_sr_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64]
        L.orc_sr_uniform.restype = C.c_float
        L.orc_quantize.argtypes = [_P, C.c_int64, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int64, _P,
                                   _P, _P, _P]
        L.orc_exp_p.argtypes = [C.c_float]
        L.orc_exp_p.restype = C.c_float
        L.orc_error_term.argtypes = [C.c_float, C.c_float]
        L.orc_error_term.restype = C.c_float
        L.orc_error_x.argtypes = [_P, _P, C.c_float, C.c_int64]
        L.orc_error_x.restype = C.c_double
        L.orc_select_bits.argtypes = [_P, C.c_int64, C.c_float, C.c_int, C.c_int, _P, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int)]
        L.orc_sddmm_add.argtypes = [C.POINTER(Graph), C.c_int, QRef, QRef, C.c_float, _P, _P]
        L.orc_edge_softmax.argtypes = [C.POINTER(Graph), C.c_int, _P, _P, _P, _P]
        L.orc_spmm_alpha.argtypes = [C.POINTER(Graph), C.c_int, C.c_int, C.c_int, _P, QRef, _P]
        L.orc_sddmm_dot.argtypes = [C.POINTER(Graph), C.c_int, C.c_int, QRef, QRef, _P]
        L.orc_softmax_bwd.argtypes = [C.POINTER(Graph), C.c_int, _P, _P, _P, C.c_float, _P, _P, _P]
        L.orc_edge_sum.argtypes = [C.POINTER(Graph), C.c_int, C.c_int, _P, _P]
        L.orc_spmm_sum.argtypes = [C.POINTER(Graph), C.c_int, C.c_int, QRef, _P, _P]
        L.orc_spmm_q8.argtypes = [C.POINTER(Graph), C.c_int, C.c_int, C.c_int, _P, C.c_float, _P, C.c_float, _P, _P]
        L.orc_gemm.argtypes = [C.c_int64, C.c_int64, C.c_int64, QRef, C.c_int64, C.c_int, QRef, C.c_int64, C.c_int,
                               _P, _P]
        L.orc_gat_fwd.argtypes = [C.POINTER(Graph), C.POINTER(Cfg), _P, _P, _P, _P, C.POINTER(FwdOut)]
        L.orc_gat_bwd.argtypes = [C.POINTER(Graph), C.POINTER(Cfg), _P, _P, _P, C.POINTER(FwdOut), _P, _P,
                                  C.POINTER(BwdOut)]
        L.orc_gcn_fwd.argtypes = [C.POINTER(Graph), C.POINTER(Cfg), _P, _P, C.POINTER(GcnFwdOut)]
        L.orc_gcn_bwd.argtypes = [C.POINTER(Graph), C.POINTER(Cfg), _P, _P, C.POINTER(GcnFwdOut), _P,
                                  C.POINTER(GcnBwdOut)]
        L.orc_sgemm.argtypes = [C.c_int64, C.c_int64, C.c_int64, _P, C.c_int64, C.c_int, _P, C.c_int64, C.c_int, _P]
        L.orc_colsum.argtypes = [_P, C.c_int64, C.c_int64, _P]
        L.orc_bias_relu_fwd.argtypes = [_P, _P, C.c_int64, C.c_int64, _P, _P]
        L.orc_bias_relu_bwd.argtypes = [_P, _P, C.c_int64, C.c_int64, _P, _P, _P]
        L.orc_gat_out_fwd.argtypes = [C.POINTER(Graph), C.POINTER(OutCfg), _P, _P, _P, _P, _P,
                                      C.POINTER(OutFwdOut)]
        L.orc_gat_out_bwd.argtypes = [C.POINTER(Graph), C.POINTER(OutCfg), _P, _P, _P, _P, C.POINTER(OutFwdOut),
                                      _P, C.POINTER(OutBwdOut)]
        L.orc_cross_entropy.argtypes = [_P, _P, C.c_int64, C.c_int32, C.c_int64, _P, _P, _P]
        L.orc_sgd.argtypes = [_P, _P, C.c_int64, C.c_float]
        L.orc_spmm_alpha_unit.argtypes = [C.POINTER(Graph), C.c_int, C.c_int, _P, _P]
        L.orc_gcn_out_fwd.argtypes = [C.POINTER(Graph), C.c_int, C.c_int, _P, _P, _P, C.POINTER(GcnOutFwdOut)]
        L.orc_gcn_out_bwd.argtypes = [C.POINTER(Graph), C.c_int, C.c_int, _P, _P, _P, C.POINTER(GcnOutBwdOut)]
        L.orc_num_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class OracleError(RuntimeError):
    pass


def _check(st):
    if st != 0:
        raise OracleError(f"oracle status {st}")


def set_threads(t: int):
    lib().orc_set_threads(int(t))


def num_threads() -> int:
    return lib().orc_num_threads()


# ------------------------------------------------------------------ primitives
def philox(ctr, key):
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def sr_uniform(seed, step, tag, g) -> float:
    return float(lib().orc_sr_uniform(seed, step, tag, g))


def quantize(x, bits=8, seed=0, step=0, tag=0, g0=0, amax=None):
    x = _c(x, np.float32)
    q = np.zeros(x.shape, np.int8)
    s = np.zeros(1, np.float32)
    am = np.zeros(1, np.float32)
    amin = None if amax is None else np.array([amax], np.float32)
    st = lib().orc_quantize(_p(x), x.size, bits, seed, step, tag, g0, _p(amin), _p(q), _p(s), _p(am))
    _check(st)
    return q, np.float32(s[0]), np.float32(am[0])


def error_term(x, xh) -> np.float32:
    return np.float32(lib().orc_error_term(float(np.float32(x)), float(np.float32(xh))))


def error_x(x, q, s) -> float:
    """Error_X (Eq.4, reading A24 denominator) of codes q with scale s against x."""
    x = _c(x, np.float32)
    q = _c(q, np.int8)
    return float(lib().orc_error_x(_p(x), _p(q), float(s), x.size))


def select_bits(x, threshold=0.3, bmin=2, bmax=8):
    """(bits, errs[bmin..bmax], none) with nearest rounding (reading R31)."""
    x = _c(x, np.float32)
    errs = np.zeros(bmax - bmin + 1, np.float64)
    bits = C.c_int(0)
    none = C.c_int(0)
    _check(lib().orc_select_bits(_p(x), x.size, float(threshold), bmin, bmax, _p(errs), C.byref(bits),
                                 C.byref(none)))
    return bits.value, errs, bool(none.value)


def exp_p(x: float) -> np.float32:
    return np.float32(lib().orc_exp_p(float(np.float32(x))))


def graph_struct(g, chunk=256):
    in_ptr = _c(g.in_ptr, np.int64)
    in_src = _c(g.in_src, np.int32)
    gs = Graph(g.n, in_src.shape[0], in_ptr.ctypes.data, in_src.ctypes.data, chunk)
    gs._keep = (in_ptr, in_src)
    return gs


def qref(q=None, v=None, s=1.0):
    """Codes q (int8) with scale s, or bypass fp32 values v (s = 1)."""
    if q is not None:
        q = _c(q, np.int8)
        r = QRef(q.ctypes.data, None, float(s))
        r._keep = q
    else:
        v = _c(v, np.float32)
        r = QRef(None, v.ctypes.data, float(s))
        r._keep = v
    return r


def sddmm_add(g, heads, S: QRef, D: QRef, slope, chunk=256):
    gs = graph_struct(g, chunk)
    e_pre = np.zeros((g.e, heads), np.float32)
    el = np.zeros((g.e, heads), np.float32)
    lib().orc_sddmm_add(C.byref(gs), heads, S, D, slope, _p(e_pre), _p(el))
    return e_pre, el


def edge_softmax(g, heads, el, chunk=256):
    gs = graph_struct(g, chunk)
    el = _c(el, np.float32)
    m = np.zeros((g.n, heads), np.float32)
    den = np.zeros((g.n, heads), np.float32)
    alpha = np.zeros((g.e, heads), np.float32)
    lib().orc_edge_softmax(C.byref(gs), heads, _p(el), _p(m), _p(den), _p(alpha))
    return m, den, alpha


def spmm_alpha(g, direction, heads, cols, alpha, X: QRef, chunk=256):
    gs = graph_struct(g, chunk)
    alpha = _c(alpha, np.float32)
    out = np.zeros((g.n, cols), np.float32)
    _check(lib().orc_spmm_alpha(C.byref(gs), direction, heads, cols, _p(alpha), X, _p(out)))
    return out


def sddmm_dot(g, heads, cols, A: QRef, B: QRef, chunk=256):
    gs = graph_struct(g, chunk)
    out = np.zeros((g.e, heads), np.float32)
    lib().orc_sddmm_dot(C.byref(gs), heads, cols, A, B, _p(out))
    return out


def softmax_bwd(g, heads, alpha, dalpha, e_pre, slope, chunk=256):
    gs = graph_struct(g, chunk)
    alpha, dalpha, e_pre = (_c(a, np.float32) for a in (alpha, dalpha, e_pre))
    P = np.zeros((g.n, heads), np.float32)
    dE = np.zeros((g.e, heads), np.float32)
    dEp = np.zeros((g.e, heads), np.float32)
    lib().orc_softmax_bwd(C.byref(gs), heads, _p(alpha), _p(dalpha), _p(e_pre), slope, _p(P), _p(dE), _p(dEp))
    return P, dE, dEp


def edge_sum(g, direction, heads, x, chunk=256):
    gs = graph_struct(g, chunk)
    x = _c(x, np.float32)
    out = np.zeros((g.n, heads), np.float32)
    _check(lib().orc_edge_sum(C.byref(gs), direction, heads, _p(x), _p(out)))
    return out


def spmm_q8(g, direction, heads, cols, qa, sa, qx, sx):
    """NEXT-4 int8-α SPMM (orc_spmm_q8): exact int32 sums of q_α·q_X and (float)acc · fl(s_α·s_X)."""
    gs = graph_struct(g, 256)
    qa = _c(qa, np.int8)
    qx = _c(qx, np.int8)
    oi = np.zeros((g.n, cols), np.int32)
    of = np.zeros((g.n, cols), np.float32)
    _check(lib().orc_spmm_q8(C.byref(gs), direction, heads, cols, _p(qa), C.c_float(sa), _p(qx), C.c_float(sx),
                             _p(oi), _p(of)))
    return oi, of


def spmm_sum(g, direction, cols, X: QRef, chunk=256):
    gs = graph_struct(g, chunk)
    oi = np.zeros((g.n, cols), np.int32)
    of = np.zeros((g.n, cols), np.float32)
    _check(lib().orc_spmm_sum(C.byref(gs), direction, cols, X, _p(oi), _p(of)))
    return oi, of


def gemm(A: QRef, B: QRef, M, N, K, lda, ldb, transA=False, transB=False):
    acc64 = np.zeros((M, N), np.int64)
    accf = np.zeros((M, N), np.float32)
    lib().orc_gemm(M, N, K, A, lda, int(transA), B, ldb, int(transB), _p(acc64), _p(accf))
    return acc64, accf


# ------------------------------------------------------------------ layers
def _cfg(F, H, D, slope, bits, seed, step, layer_id):
    return Cfg(F, H, D, slope, bits, seed, step, layer_id)


def gat_fwd(g, H, W, a_src, a_dst, heads, head_dim, slope=0.2, bits=8, seed=0x7A4E60, step=0, layer_id=0,
            chunk=256):
    n, F = H.shape
    HD = heads * head_dim
    E = g.e
    gs = graph_struct(g, chunk)
    cfg = _cfg(F, heads, head_dim, slope, bits, seed, step, layer_id)
    H, W, a_src, a_dst = (_c(a, np.float32) for a in (H, W, a_src, a_dst))
    o = dict(qH=np.zeros((n, F), np.int8), sH=np.zeros(1, np.float32), qW=np.zeros((F, HD), np.int8),
             sW=np.zeros(1, np.float32), maxacc=np.zeros(1, np.int32), Hp=np.zeros((n, HD), np.float32),
             S=np.zeros((n, heads), np.float32), Dd=np.zeros((n, heads), np.float32),
             qHp=np.zeros((n, HD), np.int8), sHp=np.zeros(1, np.float32), qS=np.zeros((n, heads), np.int8),
             sS=np.zeros(1, np.float32), qD=np.zeros((n, heads), np.int8), sD=np.zeros(1, np.float32),
             e_pre=np.zeros((E, heads), np.float32), alpha=np.zeros((E, heads), np.float32),
             m=np.zeros((n, heads), np.float32), den=np.zeros((n, heads), np.float32),
             Hout=np.zeros((n, HD), np.float32), amax_out=np.zeros(1, np.float32))
    st = FwdOut(*[_p(o[f]) for f in _FWD_FIELDS])
    _check(lib().orc_gat_fwd(C.byref(gs), C.byref(cfg), _p(H), _p(W), _p(a_src), _p(a_dst), C.byref(st)))
    o["_struct"] = st
    o["_cfg"] = dict(F=F, heads=heads, head_dim=head_dim, slope=slope, bits=bits, seed=seed, step=step,
                     layer_id=layer_id, chunk=chunk)
    return o


def gat_bwd(g, fwd, H, W, a_src, a_dst, dHout):
    c = fwd["_cfg"]
    n, F = H.shape
    heads, hd = c["heads"], c["head_dim"]
    HD = heads * hd
    E = g.e
    gs = graph_struct(g, c["chunk"])
    cfg = _cfg(F, heads, hd, c["slope"], c["bits"], c["seed"], c["step"], c["layer_id"])
    H, W, a_src, a_dst, dHout = (_c(a, np.float32) for a in (H, W, a_src, a_dst, dHout))
    o = dict(qG=np.zeros((n, HD), np.int8), sG=np.zeros(1, np.float32), dalpha=np.zeros((E, heads), np.float32),
             P=np.zeros((n, heads), np.float32), dE=np.zeros((E, heads), np.float32),
             dE_pre=np.zeros((E, heads), np.float32), dD=np.zeros((n, heads), np.float32),
             dS=np.zeros((n, heads), np.float32), dHp_agg=np.zeros((n, HD), np.float32),
             dHp=np.zeros((n, HD), np.float32), da_src=np.zeros(HD, np.float32), da_dst=np.zeros(HD, np.float32),
             da_src_abs=np.zeros(HD, np.float32), da_dst_abs=np.zeros(HD, np.float32),
             qdHp=np.zeros((n, HD), np.int8), sdHp=np.zeros(1, np.float32), dH=np.zeros((n, F), np.float32),
             dW=np.zeros((F, HD), np.float32))
    st = BwdOut(*[_p(o[f]) for f in _BWD_FIELDS])
    _check(lib().orc_gat_bwd(C.byref(gs), C.byref(cfg), _p(W), _p(a_src), _p(a_dst), C.byref(fwd["_struct"]),
                             _p(H), _p(dHout), C.byref(st)))
    return o


def gcn_fwd(g, X, W, bits=8, seed=0x7A4E60, step=0, layer_id=0, chunk=256):
    n, F = X.shape
    O = W.shape[1]
    gs = graph_struct(g, chunk)
    cfg = _cfg(F, 1, O, 0.0, bits, seed, step, layer_id)
    X, W = _c(X, np.float32), _c(W, np.float32)
    o = dict(qX=np.zeros((n, F), np.int8), sX=np.zeros(1, np.float32), qW=np.zeros((F, O), np.int8),
             sW=np.zeros(1, np.float32), Ys=np.zeros((n, O), np.float32), qYs=np.zeros((n, O), np.int8),
             sYs=np.zeros(1, np.float32), ia=np.zeros((n, O), np.int32), out=np.zeros((n, O), np.float32))
    st = GcnFwdOut(*[_p(o[f]) for f in _GCN_FWD_FIELDS])
    _check(lib().orc_gcn_fwd(C.byref(gs), C.byref(cfg), _p(X), _p(W), C.byref(st)))
    o["_struct"] = st
    o["_cfg"] = dict(F=F, O=O, bits=bits, seed=seed, step=step, layer_id=layer_id, chunk=chunk)
    return o


def gcn_bwd(g, fwd, X, W, dout):
    c = fwd["_cfg"]
    n, F = X.shape
    O = c["O"]
    gs = graph_struct(g, c["chunk"])
    cfg = _cfg(F, 1, O, 0.0, c["bits"], c["seed"], c["step"], c["layer_id"])
    X, W, dout = _c(X, np.float32), _c(W, np.float32), _c(dout, np.float32)
    o = dict(Gs=np.zeros((n, O), np.float32), qGs=np.zeros((n, O), np.int8), sGs=np.zeros(1, np.float32),
             ib=np.zeros((n, O), np.int32), dY=np.zeros((n, O), np.float32), qdY=np.zeros((n, O), np.int8),
             sdY=np.zeros(1, np.float32), dX=np.zeros((n, F), np.float32), dW=np.zeros((F, O), np.float32))
    st = GcnBwdOut(*[_p(o[f]) for f in _GCN_BWD_FIELDS])
    _check(lib().orc_gcn_bwd(C.byref(gs), C.byref(cfg), _p(X), _p(W), C.byref(fwd["_struct"]), _p(dout),
                             C.byref(st)))
    return o


# ------------------------------------------------------------------ NEXT-1: the training step around the layer
def sgemm(A, B, transA=False, transB=False):
    """Full-precision GEMM with the pinned K-chunked FMA order (reading R33)."""
    A, B = _c(A, np.float32), _c(B, np.float32)
    M, K = (A.shape[1], A.shape[0]) if transA else A.shape
    N = B.shape[0] if transB else B.shape[1]
    out = np.zeros((M, N), np.float32)
    lib().orc_sgemm(M, N, K, _p(A), A.shape[1], int(transA), _p(B), B.shape[1], int(transB), _p(out))
    return out


def colsum(x):
    x = _c(x, np.float32)
    out = np.zeros(x.shape[1], np.float32)
    lib().orc_colsum(_p(x), x.shape[0], x.shape[1], _p(out))
    return out


def bias_relu_fwd(x, b):
    x, b = _c(x, np.float32), _c(b, np.float32)
    a = np.zeros_like(x)
    am = np.zeros(1, np.float32)
    lib().orc_bias_relu_fwd(_p(x), _p(b), x.shape[0], x.shape[1], _p(a), _p(am))
    return a, np.float32(am[0])


def bias_relu_bwd(a, da):
    a, da = _c(a, np.float32), _c(da, np.float32)
    dx = np.zeros_like(a)
    db = np.zeros(a.shape[1], np.float32)
    am = np.zeros(1, np.float32)
    lib().orc_bias_relu_bwd(_p(a), _p(da), a.shape[0], a.shape[1], _p(dx), _p(db), _p(am))
    return dx, db, np.float32(am[0])


def gat_out_fwd(g, H, W, a_src, a_dst, bias, heads, classes, slope=0.2, chunk=256):
    """Full-precision final GAT layer with head mean and bias (reading R35)."""
    n, F = H.shape
    HC = heads * classes
    gs = graph_struct(g, chunk)
    cfg = OutCfg(F, heads, classes, slope)
    H, W, a_src, a_dst, bias = (_c(a, np.float32) for a in (H, W, a_src, a_dst, bias))
    o = dict(Hp=np.zeros((n, HC), np.float32), S=np.zeros((n, heads), np.float32),
             Dd=np.zeros((n, heads), np.float32), e_pre=np.zeros((g.e, heads), np.float32),
             alpha=np.zeros((g.e, heads), np.float32), m=np.zeros((n, heads), np.float32),
             den=np.zeros((n, heads), np.float32), agg=np.zeros((n, HC), np.float32),
             logits=np.zeros((n, classes), np.float32))
    st = OutFwdOut(*[_p(o[f]) for f in _OUT_FWD_FIELDS])
    _check(lib().orc_gat_out_fwd(C.byref(gs), C.byref(cfg), _p(H), _p(W), _p(a_src), _p(a_dst), _p(bias),
                                 C.byref(st)))
    o["_struct"] = st
    o["_cfg"] = dict(F=F, heads=heads, classes=classes, slope=slope, chunk=chunk)
    return o


def gat_out_bwd(g, fwd, H, W, a_src, a_dst, dlogits, want_dH=True):
    c = fwd["_cfg"]
    n, F = H.shape
    heads, classes = c["heads"], c["classes"]
    HC = heads * classes
    E = g.e
    gs = graph_struct(g, c["chunk"])
    cfg = OutCfg(F, heads, classes, c["slope"])
    H, W, a_src, a_dst, dlogits = (_c(a, np.float32) for a in (H, W, a_src, a_dst, dlogits))
    o = dict(db=np.zeros(classes, np.float32), G=np.zeros((n, classes), np.float32),
             dalpha=np.zeros((E, heads), np.float32), P=np.zeros((n, heads), np.float32),
             dE=np.zeros((E, heads), np.float32), dE_pre=np.zeros((E, heads), np.float32),
             dD=np.zeros((n, heads), np.float32), dS=np.zeros((n, heads), np.float32),
             dHp_agg=np.zeros((n, HC), np.float32), dHp=np.zeros((n, HC), np.float32),
             da_src=np.zeros(HC, np.float32), da_dst=np.zeros(HC, np.float32),
             da_src_abs=np.zeros(HC, np.float32), da_dst_abs=np.zeros(HC, np.float32),
             dH=np.zeros((n, F), np.float32) if want_dH else None, dW=np.zeros((F, HC), np.float32))
    st = OutBwdOut(*[_p(o[f]) for f in _OUT_BWD_FIELDS])
    _check(lib().orc_gat_out_bwd(C.byref(gs), C.byref(cfg), _p(H), _p(W), _p(a_src), _p(a_dst),
                                 C.byref(fwd["_struct"]), _p(dlogits), C.byref(st)))
    return o


def cross_entropy(z, labels, n_lab=None):
    """(loss, dz, row_loss) over rows with label >= 0 (reading R36)."""
    z = _c(z, np.float32)
    labels = _c(labels, np.int32)
    n, Cc = z.shape
    if n_lab is None:
        n_lab = int((labels >= 0).sum())
    dz = np.zeros_like(z)
    rl = np.zeros(n, np.float32)
    loss = C.c_double(0.0)
    _check(lib().orc_cross_entropy(_p(z), _p(labels), n, Cc, n_lab, _p(rl), C.byref(loss), _p(dz)))
    return loss.value, dz, rl


def sgd(w, g, lr):
    """Returns W − lr·∂W (Eq.6: the FP32 master takes the FP32 gradient)."""
    w = _c(w, np.float32).copy()
    g = _c(g, np.float32)
    lib().orc_sgd(_p(w), _p(g), w.size, float(lr))
    return w


def gat_model_step(g, X, hidden, out, labels, lr, bits=8, seed=0x7A4E60, step=0, slope=0.2, chunk=256):
    """One full-batch training step of the multi-layer GAT, composed from the
    oracle's layer functions in the paper's order:

      hidden layer l = 1..L-1 (quantized, heads concatenated, layer_id = l):
          H_l = ReLU(gat_fwd(H_{l-1}) + b_l)                     (reading R34)
      final layer (FP32; heads averaged, reading R35):
          logits = gat_out_fwd(H_{L-1}) ; loss = CE(logits, labels) (R36)
      backward in reverse (the first layer's ∂H is not needed), then
      W ← W − lr·∂W for every FP32 master (Eq.6).

    hidden: list of dicts {W, a_src, a_dst, b, heads, head_dim}; out: {W, a_src, a_dst, b, heads, classes}.
    Returns dict(loss, logits, fwd/bwd records, grads, new params)."""
    hs = [np.asarray(X, np.float32)]
    fws, acts = [], []
    for l, p in enumerate(hidden, start=1):
        f = gat_fwd(g, hs[-1], p["W"], p["a_src"], p["a_dst"], p["heads"], p["head_dim"], slope=slope, bits=bits,
                    seed=seed, step=step, layer_id=l, chunk=chunk)
        a, am = bias_relu_fwd(f["Hout"], p["b"])
        fws.append(f)
        acts.append(am)
        hs.append(a)
    fo = gat_out_fwd(g, hs[-1], out["W"], out["a_src"], out["a_dst"], out["b"], out["heads"], out["classes"],
                     slope=slope, chunk=chunk)
    loss, dz, _ = cross_entropy(fo["logits"], labels)
    bo = gat_out_bwd(g, fo, hs[-1], out["W"], out["a_src"], out["a_dst"], dz, want_dH=len(hidden) > 0)
    grads = [None] * len(hidden)
    dA = bo["dH"]
    bws = [None] * len(hidden)
    for i in range(len(hidden) - 1, -1, -1):
        p = hidden[i]
        dx, db, _ = bias_relu_bwd(hs[i + 1], dA)
        b = gat_bwd(g, fws[i], hs[i], p["W"], p["a_src"], p["a_dst"], dx)
        bws[i] = b
        grads[i] = dict(W=b["dW"], a_src=b["da_src"], a_dst=b["da_dst"], b=db, da_src_abs=b["da_src_abs"],
                        da_dst_abs=b["da_dst_abs"])
        dA = b["dH"]
    ogr = dict(W=bo["dW"], a_src=bo["da_src"], a_dst=bo["da_dst"], b=bo["db"], da_src_abs=bo["da_src_abs"],
               da_dst_abs=bo["da_dst_abs"])
    new_hidden = [{**p, **{k: sgd(p[k], gr[k], lr) for k in ("W", "a_src", "a_dst", "b")}}
                  for p, gr in zip(hidden, grads)]
    new_out = {**out, **{k: sgd(out[k], ogr[k], lr) for k in ("W", "a_src", "a_dst", "b")}}
    return dict(loss=loss, logits=fo["logits"], hs=hs, fwd=fws, out_fwd=fo, out_bwd=bo, bwd=bws, grads=grads,
                out_grads=ogr, hidden=new_hidden, out=new_out)


def gather_sum(g, direction, x, chunk=256):
    """Unweighted fp32 chunked row gather (R14): in-edges (0) or out-edges (1)."""
    gs = graph_struct(g, chunk)
    x = _c(x, np.float32)
    out = np.zeros((g.n, x.shape[1]), np.float32)
    _check(lib().orc_spmm_alpha_unit(C.byref(gs), direction, x.shape[1], _p(x), _p(out)))
    return out


def gcn_out_fwd(g, X, W, bias, chunk=256):
    """Full-precision final GCN layer (R26 norms, R35 bias)."""
    n, F = X.shape
    Cc = W.shape[1]
    gs = graph_struct(g, chunk)
    X, W, bias = (_c(a, np.float32) for a in (X, W, bias))
    o = {k: np.zeros((n, Cc), np.float32) for k in ("Y", "Ys", "agg", "logits")}
    st = GcnOutFwdOut(*[_p(o[k]) for k in ("Y", "Ys", "agg", "logits")])
    _check(lib().orc_gcn_out_fwd(C.byref(gs), F, Cc, _p(X), _p(W), _p(bias), C.byref(st)))
    o["_cfg"] = dict(F=F, C=Cc, chunk=chunk)
    return o


def gcn_out_bwd(g, fwd, X, W, dlogits, want_dX=True):
    c = fwd["_cfg"]
    n, F = X.shape
    Cc = c["C"]
    gs = graph_struct(g, c["chunk"])
    X, W, dlogits = (_c(a, np.float32) for a in (X, W, dlogits))
    o = dict(db=np.zeros(Cc, np.float32), Gs=np.zeros((n, Cc), np.float32), aggb=np.zeros((n, Cc), np.float32),
             dY=np.zeros((n, Cc), np.float32), dX=np.zeros((n, F), np.float32) if want_dX else None,
             dW=np.zeros((F, Cc), np.float32))
    st = GcnOutBwdOut(*[_p(o[k]) for k in ("db", "Gs", "aggb", "dY", "dX", "dW")])
    _check(lib().orc_gcn_out_bwd(C.byref(gs), F, Cc, _p(X), _p(W), _p(dlogits), C.byref(st)))
    return o


def gcn_model_step(g, X, hidden, out, labels, lr, bits=8, seed=0x7A4E60, step=0, chunk=256):
    """One full-batch training step of a multi-layer GCN (NEXT-1): hidden layers l = 1..L-1 are the
    quantized GCN layer (orc_gcn_fwd, layer_id = l) followed by bias + ReLU (R34); the final layer is
    FP32 (gcn_out_fwd); cross-entropy (R36); backward in reverse; SGD on every FP32 master (R37).
    hidden: [{W, b}], out: {W, b}."""
    hs = [np.asarray(X, np.float32)]
    fws = []
    for l, p in enumerate(hidden, start=1):
        f = gcn_fwd(g, hs[-1], p["W"], bits=bits, seed=seed, step=step, layer_id=l, chunk=chunk)
        a, _ = bias_relu_fwd(f["out"], p["b"])
        fws.append(f)
        hs.append(a)
    fo = gcn_out_fwd(g, hs[-1], out["W"], out["b"], chunk=chunk)
    loss, dz, _ = cross_entropy(fo["logits"], labels)
    bo = gcn_out_bwd(g, fo, hs[-1], out["W"], dz, want_dX=len(hidden) > 0)
    grads = [None] * len(hidden)
    dA = bo["dX"]
    for i in range(len(hidden) - 1, -1, -1):
        dx, db, _ = bias_relu_bwd(hs[i + 1], dA)
        b = gcn_bwd(g, fws[i], hs[i], hidden[i]["W"], dx)
        grads[i] = dict(W=b["dW"], b=db)
        dA = b["dX"]
    ogr = dict(W=bo["dW"], b=bo["db"])
    new_hidden = [{**p, **{k: sgd(p[k], gr[k], lr) for k in ("W", "b")}} for p, gr in zip(hidden, grads)]
    new_out = {**out, **{k: sgd(out[k], ogr[k], lr) for k in ("W", "b")}}
    return dict(loss=loss, logits=fo["logits"], hs=hs, out_fwd=fo, out_bwd=bo, grads=grads, out_grads=ogr,
                hidden=new_hidden, out=new_out)
