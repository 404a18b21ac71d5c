"""Oracle sparse primitives vs their dense textbook definitions (§2.1):
E = G⊙(S⊕Dᵀ), α = masked softmax, H = (G⊙α)·H′, ∂H′ = (Gᵀ⊙α)·∂H, ∂α = G⊙(∂H·H′ᵀ),
∂D = (G⊙∂E)·1, ∂S = (Gᵀ⊙∂E)·1, and the integer GCN aggregation.  float64 dense
numpy / torch autograd are the independent references (SPEC S:575 idea:
random graphs with V <= 64, tolerance 1e-5).
"""
import numpy as np
import pytest
import torch

from paper_2308_00890_b200 import inputs

CASES = [(n, draws, seed) for seed, (n, draws) in enumerate([(5, 6), (17, 40), (33, 90), (64, 256), (64, 20),
                                                            (48, 300), (9, 0), (40, 120)])]


def dense_mask(gr):
    G = np.zeros((gr.n, gr.n), bool)      # G[dst, src]
    G[gr.in_dst(), gr.in_src] = True
    return G


@pytest.fixture(params=CASES, ids=lambda c: f"n{c[0]}d{c[1]}s{c[2]}")
def case(request):
    n, draws, seed = request.param
    gr = inputs.random_graph(n, draws, seed=seed, self_loops=(seed % 3 != 2))
    rng = np.random.default_rng(100 + seed)
    return gr, rng


def test_sddmm_add(orc, case):
    gr, rng = case
    H = 3
    S = rng.standard_normal((gr.n, H)).astype(np.float32)
    D = rng.standard_normal((gr.n, H)).astype(np.float32)
    e_pre, el = orc.sddmm_add(gr, H, orc.qref(v=S), orc.qref(v=D), 0.2)
    dense = S[None, :, :].astype(np.float64) + D[:, None, :]          # [dst, src, h]
    ref = dense[gr.in_dst(), gr.in_src]
    assert np.allclose(e_pre, ref, rtol=1e-6, atol=1e-6)
    assert np.allclose(el, np.where(ref > 0, ref, 0.2 * ref), rtol=1e-6, atol=1e-6)


def test_edge_softmax_and_spmm(orc, case):
    gr, rng = case
    H, hd = 2, 5
    el = (rng.standard_normal((gr.e, H)) * 3).astype(np.float32)
    m, den, alpha = orc.edge_softmax(gr, H, el, chunk=4)
    G = dense_mask(gr)
    A = np.full((gr.n, gr.n, H), -np.inf)
    A[gr.in_dst(), gr.in_src] = el
    with np.errstate(invalid="ignore"):
        mx = A.max(axis=1, keepdims=True)
        ex = np.where(G[:, :, None], np.exp(A - np.where(np.isfinite(mx), mx, 0)), 0.0)
        sm = ex / ex.sum(axis=1, keepdims=True)
    ref = sm[gr.in_dst(), gr.in_src]
    assert np.allclose(alpha, ref, rtol=1e-5, atol=1e-6)
    # Σα = 1 per non-empty row
    deg = np.diff(gr.in_ptr)
    sums = np.zeros((gr.n, H))
    np.add.at(sums, gr.in_dst(), alpha)
    assert np.allclose(sums[deg > 0], 1.0, atol=1e-6)
    assert np.all(den[deg == 0] == 0) and np.all(m[deg == 0] == 0)
    # ⑤ H_out = (G⊙α)·X per head, and ⑤′ (Gᵀ⊙α)·X
    X = rng.standard_normal((gr.n, H * hd)).astype(np.float32)
    out = orc.spmm_alpha(gr, 0, H, H * hd, alpha, orc.qref(v=X), chunk=3)
    outr = orc.spmm_alpha(gr, 1, H, H * hd, alpha, orc.qref(v=X), chunk=3)
    Wd = np.zeros((gr.n, gr.n, H))
    Wd[gr.in_dst(), gr.in_src] = alpha
    for h in range(H):
        Xh = X[:, h * hd:(h + 1) * hd].astype(np.float64)
        assert np.allclose(out[:, h * hd:(h + 1) * hd], Wd[:, :, h] @ Xh, rtol=1e-5, atol=1e-5)
        assert np.allclose(outr[:, h * hd:(h + 1) * hd], Wd[:, :, h].T @ Xh, rtol=1e-5, atol=1e-5)


def test_sddmm_dot_quantized_and_bypass(orc, case):
    gr, rng = case
    H, hd = 2, 7
    A = rng.integers(-127, 128, size=(gr.n, H * hd)).astype(np.int8)
    B = rng.integers(-127, 128, size=(gr.n, H * hd)).astype(np.int8)
    sa, sb = np.float32(0.013), np.float32(0.77)
    out = orc.sddmm_dot(gr, H, H * hd, orc.qref(q=A, s=sa), orc.qref(q=B, s=sb))
    for h in range(H):
        dense = A[:, h * hd:(h + 1) * hd].astype(np.int64) @ B[:, h * hd:(h + 1) * hd].astype(np.int64).T
        ref = dense[gr.in_dst(), gr.in_src].astype(np.float32) * np.float32(sa * sb)
        assert np.array_equal(out[:, h], ref)          # exact: (float)int * (sA*sB)
    Af, Bf = A.astype(np.float32) * 0.1, B.astype(np.float32) * 0.2
    out = orc.sddmm_dot(gr, H, H * hd, orc.qref(v=Af), orc.qref(v=Bf))
    for h in range(H):
        dense = Af[:, h * hd:(h + 1) * hd].astype(np.float64) @ Bf[:, h * hd:(h + 1) * hd].astype(np.float64).T
        assert np.allclose(out[:, h], dense[gr.in_dst(), gr.in_src], rtol=1e-6, atol=1e-6)


def test_softmax_backward_and_incidence(orc, case):
    gr, rng = case
    H = 3
    e_pre = rng.standard_normal((gr.e, H)).astype(np.float32)
    slope = 0.2
    el = np.where(e_pre > 0, e_pre, e_pre * np.float32(slope)).astype(np.float32)
    _, _, alpha = orc.edge_softmax(gr, H, el, chunk=5)
    dalpha = rng.standard_normal((gr.e, H)).astype(np.float32)
    P, dE, dEp = orc.softmax_bwd(gr, H, alpha, dalpha, e_pre, slope, chunk=5)
    # autograd reference of per-destination softmax + LeakyReLU
    dst = torch.from_numpy(gr.in_dst().astype(np.int64))
    ep = torch.tensor(e_pre, dtype=torch.float64, requires_grad=True)
    elt = torch.nn.functional.leaky_relu(ep, slope)
    mx = torch.full((gr.n, H), -torch.inf, dtype=torch.float64).scatter_reduce(
        0, dst[:, None].expand(-1, H), elt, "amax", include_self=True)
    ex = torch.exp(elt - mx[dst])
    den = torch.zeros((gr.n, H), dtype=torch.float64).index_add(0, dst, ex)
    a = ex / den[dst]
    a.backward(torch.tensor(dalpha, dtype=torch.float64))
    assert np.allclose(dEp, ep.grad.numpy(), rtol=1e-4, atol=1e-5)
    # incidence SPMMs vs dense incidence matrices
    Iin = np.zeros((gr.n, gr.e))
    Iin[gr.in_dst(), np.arange(gr.e)] = 1
    Iout = np.zeros((gr.n, gr.e))
    Iout[gr.in_src, np.arange(gr.e)] = 1
    dD = orc.edge_sum(gr, 0, H, dEp, chunk=2)
    dS = orc.edge_sum(gr, 1, H, dEp, chunk=2)
    assert np.allclose(dD, Iin @ dEp.astype(np.float64), rtol=1e-5, atol=1e-6)
    assert np.allclose(dS, Iout @ dEp.astype(np.float64), rtol=1e-5, atol=1e-6)


def test_int_spmm(orc, case):
    gr, rng = case
    cols = 9
    X = rng.integers(-127, 128, size=(gr.n, cols)).astype(np.int8)
    G = dense_mask(gr).astype(np.int64)
    ia, _ = orc.spmm_sum(gr, 0, cols, orc.qref(q=X))
    ib, _ = orc.spmm_sum(gr, 1, cols, orc.qref(q=X))
    assert np.array_equal(ia, G @ X.astype(np.int64))
    assert np.array_equal(ib, G.T @ X.astype(np.int64))


def test_chunking_changes_only_rounding(orc):
    gr = inputs.random_graph(64, 2000, seed=5)
    rng = np.random.default_rng(0)
    el = rng.standard_normal((gr.e, 2)).astype(np.float32)
    _, den1, a1 = orc.edge_softmax(gr, 2, el, chunk=1 << 30)
    _, den2, a2 = orc.edge_softmax(gr, 2, el, chunk=3)
    assert np.allclose(den1, den2, rtol=1e-6)
    assert np.allclose(a1, a2, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("heads,hd", [(1, 5), (2, 4), (4, 3)])
def test_spmm_q8_dense(orc, case, heads, hd):
    """NEXT-4 int8-α SPMM vs the dense product: out_i32 = (G ⊙ q_α)·q_X per head (int64 brute force, exact), in
    both directions (dir 1 = the reversed graph, α taken at each edge's in-CSR slot), and the float output
    = (float)acc · fl(s_α·s_X)."""
    gr, rng = case
    cols = heads * hd
    qa = rng.integers(-127, 128, size=(gr.e, heads)).astype(np.int8)
    qx = rng.integers(-127, 128, size=(gr.n, cols)).astype(np.int8)
    sa, sx = np.float32(0.0071), np.float32(0.013)
    dst, src = gr.in_dst(), gr.in_src
    for direction in (0, 1):
        ref = np.zeros((gr.n, cols), np.int64)
        for h in range(heads):
            A = np.zeros((gr.n, gr.n), np.int64)          # A[row, other endpoint] = q_α of the edge
            if direction == 0:
                A[dst, src] = qa[:, h]
            else:
                A[src, dst] = qa[:, h]
            ref[:, h * hd:(h + 1) * hd] = A @ qx[:, h * hd:(h + 1) * hd].astype(np.int64)
        oi, of = orc.spmm_q8(gr, direction, heads, cols, qa, sa, qx, sx)
        assert np.array_equal(oi.astype(np.int64), ref)
        assert np.array_equal(of, ref.astype(np.float32) * np.float32(sa * sx))
