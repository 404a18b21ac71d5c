"""GPU parity of the libtango primitives against the CPU oracle (called through the C ABI).

Bit-exact for int8 codes, integer accumulators and every fp32 value the oracle pins
(DESIGN.md §2 readings R1-R14); ragged sizes span several tiles plus a tail.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2308_00890_b200 import inputs  # noqa: E402


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_00890_b200 import tango
    tango.load()
    return tango


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("rows,cols,row0", [(1, 1, 0), (7, 13, 0), (333, 100, 5), (1000, 512, 0), (4097, 602, 17),
                                            (64, 1433, 0)])
def test_quantize_parity(T, orc, rows, cols, row0):
    rng = np.random.default_rng(rows + cols)
    x = (rng.standard_normal((rows, cols)) * rng.uniform(0.01, 10)).astype(np.float32)
    seed, step, tag = 0x7A4E60, 5, 0x103
    q, s, amax = T.quantize(cu(x), bits=8, seed=seed, step=step, tag=tag, global_row0=row0)
    torch.cuda.synchronize()
    qo, so, ao = orc.quantize(x, 8, seed=seed, step=step, tag=tag, g0=row0 * cols)
    qg = q.cpu().numpy()
    assert np.array_equal(qg[:, :cols], qo)
    assert np.all(qg[:, cols:] == 0)
    assert s.item() == so and amax.item() == ao


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quantize_bits_and_hint(T, orc, bits):
    x = np.random.default_rng(1).standard_normal((300, 64)).astype(np.float32)
    hint = cu(np.array([7.5], np.float32))
    q, s, amax = T.quantize(cu(x), bits=bits, seed=3, step=1, tag=9, amax_hint=hint)
    qo, so, _ = orc.quantize(x, bits, seed=3, step=1, tag=9, amax=np.float32(7.5))
    assert np.array_equal(q.cpu().numpy()[:, :64], qo) and s.item() == so


def test_quantize_zero_and_nonfinite(T):
    q, s, amax = T.quantize(torch.zeros((5, 32), device="cuda"))
    assert s.item() == 1.0 and amax.item() == 0.0 and int(q.abs().max()) == 0
    x = torch.ones((10, 32), device="cuda")
    x[3, 4] = float("nan")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    T.quantize(x, status=st)
    assert int(st.item()) == 4


def test_quantize_bad_args(T):
    with pytest.raises(T.TangoError):
        T.quantize(torch.ones((4, 32), device="cuda"), bits=9)


def _rand_i8(rng, shape):
    return rng.integers(-127, 128, size=shape).astype(np.int8)


def _pad(a, ld):
    out = np.zeros((a.shape[0], ld), np.int8)
    out[:, :a.shape[1]] = a
    return out


@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (300, 512, 128), (1000, 96, 100), (257, 512, 602),
                                   (129, 1440, 512), (5, 32, 1433)])
def test_gemm_kmajor(T, M, N, K):
    rng = np.random.default_rng(M * 7 + N + K)
    A = _rand_i8(rng, (M, K))
    Bt = _rand_i8(rng, (N, K))
    ld = (K + 31) // 32 * 32
    sA, sB = cu(np.array([0.0123], np.float32)), cu(np.array([1.7], np.float32))
    out = T.gemm_q(cu(_pad(A, ld)), sA, T.TANGO_K_MAJOR, cu(_pad(Bt, ld)), sB, T.TANGO_K_MAJOR, M, N, K,
                   want=("f32", "i32"))
    ref = A.astype(np.int64) @ Bt.astype(np.int64).T
    assert np.array_equal(out["i32"].cpu().numpy(), ref)
    s = np.float32(np.float32(0.0123) * np.float32(1.7))
    assert np.array_equal(out["f32"].cpu().numpy(), ref.astype(np.float32) * s)


@pytest.mark.parametrize("M,N,K", [(128, 512, 1000), (100, 512, 4097), (602, 256, 300), (16, 64, 130000),
                                   (128, 128, 300_000)])
def test_gemm_mnmajor_splitk(T, M, N, K):
    # ∂W = Hᵀ·∂H′: both operands stored [K][ld] (MN-major), int64 split-K reduction (reading R27)
    rng = np.random.default_rng(M + N + K)
    A = _rand_i8(rng, (K, M))
    B = _rand_i8(rng, (K, N))
    lda, ldb = (M + 31) // 32 * 32, (N + 31) // 32 * 32
    sA, sB = cu(np.array([0.5], np.float32)), cu(np.array([0.25], np.float32))
    out = T.gemm_q(cu(_pad(A, lda)), sA, T.TANGO_MN_MAJOR, cu(_pad(B, ldb)), sB, T.TANGO_MN_MAJOR, M, N, K,
                   want=("i64", "f32"))
    ref = A.astype(np.int64).T @ B.astype(np.int64)
    assert np.array_equal(out["i64"].cpu().numpy(), ref)
    assert np.array_equal(out["f32"].cpu().numpy(), ref.astype(np.float32) * np.float32(0.125))


def test_gemm_mixed_layouts(T):
    rng = np.random.default_rng(5)
    M, N, K = 200, 160, 256
    A = _rand_i8(rng, (M, K))
    B = _rand_i8(rng, (K, N))
    one = cu(np.array([1.0], np.float32))
    ref = A.astype(np.int64) @ B.astype(np.int64)
    o1 = T.gemm_q(cu(A), one, T.TANGO_K_MAJOR, cu(B), one, T.TANGO_MN_MAJOR, M, N, K, want=("i32",))
    o2 = T.gemm_q(cu(_pad(np.ascontiguousarray(A.T), 224)), one, T.TANGO_MN_MAJOR, cu(np.ascontiguousarray(B.T)), one,
                  T.TANGO_K_MAJOR, M, N, K, want=("i32",))
    assert np.array_equal(o1["i32"].cpu().numpy(), ref)
    assert np.array_equal(o2["i32"].cpu().numpy(), ref)


GRAPHS = [("toy", None), ("c0b", (64, 256, 0)), ("noself", (200, 500, 3)), ("mid", (3000, 30000, 4))]


def make_graph(spec):
    name, args = spec
    if name == "toy":
        return inputs.toy_graph()
    n, d, s = args
    return inputs.random_graph(n, d, seed=s, self_loops=(name != "noself"))


@pytest.mark.parametrize("spec", GRAPHS, ids=[g[0] for g in GRAPHS])
@pytest.mark.parametrize("chunk", [3, 256])
def test_sparse_primitives_parity(T, orc, spec, chunk):
    gr = make_graph(spec)
    dg = T.DeviceGraph(gr, chunk=chunk)
    rng = np.random.default_rng(gr.n)
    H = 2
    qS = _rand_i8(rng, (gr.n, H)); qD = _rand_i8(rng, (gr.n, H))
    sS, sD = np.float32(0.031), np.float32(0.017)
    e_pre, el = T.sddmm_add(dg, cu(qS), cu(np.array([sS])), cu(qD), cu(np.array([sD])), H, 0.2)
    oe, oel = orc.sddmm_add(gr, H, orc.qref(q=qS, s=sS), orc.qref(q=qD, s=sD), 0.2, chunk=chunk)
    assert np.array_equal(e_pre.cpu().numpy(), oe) and np.array_equal(el.cpu().numpy(), oel)
    m, den, alpha = T.edge_softmax(dg, H, el)
    om, oden, oa = orc.edge_softmax(gr, H, oel, chunk=chunk)
    assert np.array_equal(alpha.cpu().numpy(), oa)
    assert np.array_equal(m.cpu().numpy(), om) and np.array_equal(den.cpu().numpy(), oden)
    cols = 64
    qX = _rand_i8(rng, (gr.n, cols))
    sX = np.float32(0.02)
    for direction in (0, 1):
        out, _ = T.spmm(dg, direction, cu(qX), cu(np.array([sX])), cols, H, edge_w=alpha)
        ref = orc.spmm_alpha(gr, direction, H, cols, oa, orc.qref(q=qX, s=sX), chunk=chunk)
        assert np.array_equal(out.cpu().numpy(), ref)
        out, oi = T.spmm(dg, direction, cu(qX), cu(np.array([sX])), cols, H)
        ri, rf = orc.spmm_sum(gr, direction, cols, orc.qref(q=qX, s=sX))
        assert np.array_equal(oi.cpu().numpy(), ri)
    qA = _rand_i8(rng, (gr.n, cols)); qB = _rand_i8(rng, (gr.n, cols))
    dal, acc = T.sddmm_dot(dg, cu(qA), cu(np.array([np.float32(0.5)])), cu(qB), cu(np.array([np.float32(0.01)])),
                           H, cols)
    ref = orc.sddmm_dot(gr, H, cols, orc.qref(q=qA, s=np.float32(0.5)), orc.qref(q=qB, s=np.float32(0.01)))
    assert np.array_equal(dal.cpu().numpy(), ref)
    dalpha = rng.standard_normal((gr.e, H)).astype(np.float32)
    P, dEp = T.softmax_bwd(dg, H, alpha, cu(dalpha), e_pre, 0.2)
    oP, _, odEp = orc.softmax_bwd(gr, H, oa, dalpha, oe, 0.2, chunk=chunk)
    assert np.array_equal(P.cpu().numpy(), oP) and np.array_equal(dEp.cpu().numpy(), odEp)
    for direction in (0, 1):
        s = T.edge_sum(dg, direction, H, dEp)
        assert np.array_equal(s.cpu().numpy(), orc.edge_sum(gr, direction, H, odEp, chunk=chunk))


# Incidence SPMM ③′/③″ at the paper's edge-feature widths 4-20, plus widths
# past one warp (33, 300) and chunk sizes that cut hub rows into many canonical chunks; C_E = 1 with F = 300
# (13 partial slots per batch) forces the window-by-window fold of a row with more chunks than a batch.
ES_GRAPHS = [("toy", None), ("noself", (200, 500, 3)), ("hub", None)]


def _es_graph(name):
    if name == "hub":   # power-law with hub rows of several hundred edges, plus empty rows
        return inputs.chung_lu_graph(3000, 40000, 2.1, seed=11, dmax=900, self_loops=False)
    return make_graph((name, dict(ES_GRAPHS)[name]))


@pytest.mark.parametrize("name", [g[0] for g in ES_GRAPHS])
@pytest.mark.parametrize("F,chunk", [(4, 256), (7, 3), (12, 64), (16, 256), (16, 5), (20, 256), (33, 7),
                                     (300, 1), (300, 256)])
def test_edge_sum_parity(T, orc, name, F, chunk):
    gr = _es_graph(name)
    dg = T.DeviceGraph(gr, chunk=chunk)
    x = np.random.default_rng(F * 1000 + chunk).standard_normal((gr.e, F)).astype(np.float32)
    xd = cu(x)
    for direction in (0, 1):
        s = T.edge_sum(dg, direction, F, xd)
        assert np.array_equal(s.cpu().numpy(), orc.edge_sum(gr, direction, F, x, chunk=chunk)), (direction, F, chunk)


# Weighted SPMM ⑤ / ⑤′ as a standalone primitive (tango_spmm_q with edge weights):
# multi-head shapes of P:1186-1189, ragged column passes, D not a multiple of 4, byte-strided rows (ld % 4 != 0),
# plus the optional per-row scale and amax(|out|) of §8(b).
@pytest.mark.parametrize("name", ["noself", "hub"])
@pytest.mark.parametrize("H,D,ld,chunk", [(4, 128, 512, 256), (2, 48, 96, 7), (2, 300, 608, 64), (1, 37, 37, 3),
                                          (3, 5, 16, 256), (2, 128, 256, 1)])
def test_spmm_weighted_parity(T, orc, name, H, D, ld, chunk):
    gr = _es_graph(name)
    dg = T.DeviceGraph(gr, chunk=chunk)
    rng = np.random.default_rng(H * 100 + D)
    cols = H * D
    qX = _rand_i8(rng, (gr.n, ld))
    sX = np.float32(0.0173)
    w = rng.random((gr.e, H)).astype(np.float32)
    rs = rng.random(gr.n).astype(np.float32) + np.float32(0.5)
    for direction in (0, 1):
        ref = orc.spmm_alpha(gr, direction, H, cols, w, orc.qref(q=qX[:, :cols], s=sX), chunk=chunk)
        out, _ = T.spmm(dg, direction, cu(qX), cu(np.array([sX])), cols, H, edge_w=cu(w))
        assert np.array_equal(out.cpu().numpy(), ref), direction
        amax = torch.zeros(1, device="cuda")
        out2, _ = T.spmm(dg, direction, cu(qX), cu(np.array([sX])), cols, H, edge_w=cu(w), row_scale=cu(rs),
                         amax_out=amax)
        ref2 = ref * rs[:, None]            # one more fp32 rn multiply per element
        assert np.array_equal(out2.cpu().numpy(), ref2), direction
        assert amax.item() == np.abs(ref2).max()


def test_spmm_unweighted_rowscale_amax(T, orc):
    gr = _es_graph("hub")
    dg = T.DeviceGraph(gr)
    rng = np.random.default_rng(5)
    cols = 64
    qX = _rand_i8(rng, (gr.n, cols))
    sX = np.float32(0.02)
    rs = rng.random(gr.n).astype(np.float32)
    for direction in (0, 1):
        ri, rf = orc.spmm_sum(gr, direction, cols, orc.qref(q=qX, s=sX))
        amax = torch.zeros(1, device="cuda")
        out, oi = T.spmm(dg, direction, cu(qX), cu(np.array([sX])), cols, 1, row_scale=cu(rs), amax_out=amax)
        assert np.array_equal(oi.cpu().numpy(), ri)
        ref = (rf * sX) * rs[:, None]       # orc_spmm_sum's float output is (float)Σ, before the scale
        assert np.array_equal(out.cpu().numpy(), ref)
        assert amax.item() == np.abs(ref).max()


def test_quantize_without_amax_slot(T, orc):
    """tango_quantize with amax_out = NULL: the scale word doubles as the amax scratch (no allocation)."""
    x = inputs.features(333, 100, seed=9)
    q, s, _ = T.quantize(cu(x), bits=8, ld=128, want_amax=False)
    oq, os_, _ = orc.quantize(x, bits=8)
    assert np.array_equal(q.cpu().numpy()[:, :100], oq) and s.item() == os_


# NEXT-4 int8-α SPMM (tango_spmm_q8): α codes from the SR quantizer, exact int32 sums — bit-exact vs
# orc_spmm_q8, both directions, ragged column passes (cols not a multiple of 128), hub rows split into
# chunks that add atomically (C_E = 7), heads 1/2/4.
@pytest.mark.parametrize("name", ["noself", "hub"])
@pytest.mark.parametrize("H,D,ld,chunk", [(4, 128, 512, 256), (2, 48, 96, 7), (1, 36, 40, 64), (4, 64, 256, 1)])
def test_spmm_q8_parity(T, orc, name, H, D, ld, chunk):
    gr = _es_graph(name)
    dg = T.DeviceGraph(gr, chunk=chunk)
    rng = np.random.default_rng(H * 7 + D)
    cols = H * D
    qX = _rand_i8(rng, (gr.n, ld))
    sX = np.float32(0.0173)
    alpha = rng.random((gr.e, H)).astype(np.float32)
    qa, sa, _ = T.quantize(cu(alpha), bits=8, ld=H, tag=0x55)
    qa_np, sa_np = qa.cpu().numpy(), np.float32(sa.item())
    for direction in (0, 1):
        ri, rf = orc.spmm_q8(gr, direction, H, cols, qa_np, sa_np, qX[:, :cols], sX)
        out, oi = T.spmm_q8(dg, direction, qa, sa, cu(qX), cu(np.array([sX])), cols, H)
        assert np.array_equal(oi.cpu().numpy(), ri), direction
        assert np.array_equal(out.cpu().numpy(), rf), direction


def test_spmm_q8_validation(T):
    gr = _es_graph("noself")
    dg = T.DeviceGraph(gr)
    qa = torch.zeros((gr.e, 2), dtype=torch.int8, device="cuda")
    s = torch.ones(1, device="cuda")
    qX = torch.zeros((gr.n, 12), dtype=torch.int8, device="cuda")
    with pytest.raises(T.TangoError):          # D = 6: a lane's 4 columns would straddle two heads
        T.spmm_q8(dg, 0, qa, s, qX, s, 12, 2)


def test_nvtx_ranges_do_not_change_results(T, orc):
    """Tracing: with NVTX ranges on (one per library launch) the kernels run unchanged."""
    x = inputs.features(100, 64, seed=4)
    T.nvtx_enable(True)
    try:
        q, s, _ = T.quantize(cu(x), bits=8, ld=64)
    finally:
        T.nvtx_enable(False)
    oq, os_, _ = orc.quantize(x, bits=8)
    assert np.array_equal(q.cpu().numpy(), oq) and s.item() == os_
