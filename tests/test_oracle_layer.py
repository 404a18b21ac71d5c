"""Oracle GAT / GCN layers vs fp64 torch autograd of the textbook layers.

Bypass mode (bits=0) turns quantization off, so the oracle's hand-derived
backward must agree with autograd of the plain forward
to fp32 rounding: this catches a dropped term, a wrong sign, a wrong index or a
transposed operand anywhere in the layer.  Quantized mode is checked through
invariants that must hold exactly.
"""
import numpy as np
import pytest
import torch

from paper_2308_00890_b200 import inputs


def torch_gat(gr, H, W, a_src, a_dst, heads, hd, slope):
    n = gr.n
    src = torch.from_numpy(gr.in_src.astype(np.int64))
    dst = torch.from_numpy(gr.in_dst().astype(np.int64))
    Hp = H @ W
    Hp3 = Hp.view(n, heads, hd)
    S = (Hp3 * a_src.view(heads, hd)).sum(-1)
    D = (Hp3 * a_dst.view(heads, hd)).sum(-1)
    e = S[src] + D[dst]
    el = torch.nn.functional.leaky_relu(e, slope)
    mx = torch.full((n, heads), -torch.inf, dtype=H.dtype).scatter_reduce(
        0, dst[:, None].expand(-1, heads), el, "amax", include_self=True)
    ex = torch.exp(el - mx[dst])
    den = torch.zeros((n, heads), dtype=H.dtype).index_add(0, dst, ex)
    alpha = ex / den[dst]
    out = torch.zeros((n, heads, hd), dtype=H.dtype).index_add(0, dst, alpha[:, :, None] * Hp3[src])
    return out.reshape(n, heads * hd), dict(S=S, D=D, alpha=alpha, Hp=Hp)


def relerr(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-3)   # exact zeros (e.g. ∂a_dst on the toy) allow 1e-8 abs


@pytest.mark.parametrize("n,draws,heads,hd,F,seed", [(4, 0, 2, 2, 4, 0), (40, 100, 2, 8, 16, 1),
                                                      (64, 256, 4, 16, 16, 2), (30, 60, 1, 12, 9, 3)])
def test_gat_bypass_vs_autograd(orc, n, draws, heads, hd, F, seed):
    gr = inputs.toy_graph() if n == 4 else inputs.random_graph(n, draws, seed=seed)
    H = inputs.features(gr.n, F, seed=seed + 1)
    W, a_src, a_dst = inputs.gat_params(F, heads, hd, seed=seed + 2)
    dH = inputs.grad_out(gr.n, heads * hd, seed=seed + 3)
    slope = 0.2
    f = orc.gat_fwd(gr, H, W, a_src, a_dst, heads, hd, slope=slope, bits=0, chunk=3)
    b = orc.gat_bwd(gr, f, H, W, a_src, a_dst, dH)
    Ht = torch.tensor(H, dtype=torch.float64, requires_grad=True)
    Wt = torch.tensor(W, dtype=torch.float64, requires_grad=True)
    ast = torch.tensor(a_src, dtype=torch.float64, requires_grad=True)
    adt = torch.tensor(a_dst, dtype=torch.float64, requires_grad=True)
    out, inter = torch_gat(gr, Ht, Wt, ast, adt, heads, hd, slope)
    out.backward(torch.tensor(dH, dtype=torch.float64))
    assert relerr(f["Hout"], out.detach()) < 1e-5
    assert relerr(f["S"], inter["S"].detach()) < 1e-5
    assert relerr(f["alpha"], inter["alpha"].detach()) < 1e-5
    assert relerr(b["dH"], Ht.grad) < 1e-5
    assert relerr(b["dW"], Wt.grad) < 1e-5
    assert relerr(b["da_src"], ast.grad) < 1e-5
    assert relerr(b["da_dst"], adt.grad) < 1e-5


def torch_gcn(gr, X, W):
    n = gr.n
    src = torch.from_numpy(gr.in_src.astype(np.int64))
    dst = torch.from_numpy(gr.in_dst().astype(np.int64))
    din = torch.bincount(dst, minlength=n).double()
    dout = torch.bincount(src, minlength=n).double()
    coef = (dout[src].clamp(min=1) ** -0.5) * (din[dst].clamp(min=1) ** -0.5)   # DGL norm='both'
    Y = X @ W
    return torch.zeros((n, W.shape[1]), dtype=X.dtype).index_add(0, dst, coef[:, None] * Y[src])


@pytest.mark.parametrize("n,draws,F,O,seed", [(50, 120, 33, 16, 0), (64, 256, 16, 16, 1)])
def test_gcn_bypass_vs_autograd(orc, n, draws, F, O, seed):
    gr = inputs.random_graph(n, draws, seed=seed)
    X = inputs.features(gr.n, F, seed=seed + 1)
    W = inputs.gcn_params(F, O, seed=seed + 2)
    dout = inputs.grad_out(gr.n, O, seed=seed + 3)
    f = orc.gcn_fwd(gr, X, W, bits=0)
    b = orc.gcn_bwd(gr, f, X, W, dout)
    Xt = torch.tensor(X, dtype=torch.float64, requires_grad=True)
    Wt = torch.tensor(W, dtype=torch.float64, requires_grad=True)
    out = torch_gcn(gr, Xt, Wt)
    out.backward(torch.tensor(dout, dtype=torch.float64))
    assert relerr(f["out"], out.detach()) < 1e-5
    assert relerr(b["dX"], Xt.grad) < 1e-5
    assert relerr(b["dW"], Wt.grad) < 1e-5


@pytest.fixture(scope="module")
def qcase(orc):
    gr = inputs.random_graph(64, 256, seed=7)
    heads, hd, F = 4, 16, 16
    H = inputs.features(gr.n, F)
    W, a_src, a_dst = inputs.gat_params(F, heads, hd)
    dH = inputs.grad_out(gr.n, heads * hd)
    f = orc.gat_fwd(gr, H, W, a_src, a_dst, heads, hd, slope=0.2, bits=8, chunk=4)
    b = orc.gat_bwd(gr, f, H, W, a_src, a_dst, dH)
    return gr, heads, hd, F, H, W, a_src, a_dst, dH, f, b


def test_gat_quantized_invariants(orc, qcase):
    gr, heads, hd, F, H, W, a_src, a_dst, dH, f, b = qcase
    # amax(H′) = (float)max|acc| * (s_H*s_W) exactly (monotone rounding): s_H′ = that / 127
    amax_hp = np.float32(f["maxacc"][0]) * (f["sH"][0] * f["sW"][0])
    assert f["sHp"][0] == np.float32(amax_hp) / np.float32(127)
    assert np.abs(f["Hp"]).max() == amax_hp
    # H′ is exactly the dequantized integer product
    acc = f["qH"].astype(np.int64) @ f["qW"].astype(np.int64)
    assert np.array_equal(f["Hp"], acc.astype(np.float32) * (f["sH"][0] * f["sW"][0]))
    # codes in range
    for k in ("qH", "qW", "qHp", "qS", "qD"):
        assert np.abs(f[k].astype(np.int32)).max() <= 127
    for k in ("qG", "qdHp"):
        assert np.abs(b[k].astype(np.int32)).max() <= 127
    # caching: the quantized H, W reused by backward are the forward's (same tags) -> dW from them
    dW = (f["qH"].astype(np.int64).T @ b["qdHp"].astype(np.int64)).astype(np.float32) * (f["sH"][0] * b["sdHp"][0])
    assert np.array_equal(b["dW"], dW)
    # softmax invariants
    sums = np.zeros((gr.n, heads))
    np.add.at(sums, gr.in_dst(), f["alpha"])
    deg = np.diff(gr.in_ptr)
    assert np.allclose(sums[deg > 0], 1.0, atol=1e-6)
    single = np.repeat(deg == 1, deg)
    assert np.all(f["alpha"][single] == 1.0) and np.all(b["dE"][single] == 0.0)


def test_gat_quantized_close_to_fp32(orc, qcase):
    # int8 layer stays near the fp32 layer (loose: a few quantization steps), the accuracy premise of P:423
    gr, heads, hd, F, H, W, a_src, a_dst, dH, f, b = qcase
    f0 = orc.gat_fwd(gr, H, W, a_src, a_dst, heads, hd, slope=0.2, bits=0, chunk=4)
    b0 = orc.gat_bwd(gr, f0, H, W, a_src, a_dst, dH)
    assert relerr(f["Hout"], f0["Hout"]) < 0.05
    assert relerr(b["dH"], b0["dH"]) < 0.1
    assert relerr(b["dW"], b0["dW"]) < 0.1


def test_gat_quantized_unbiased_linear_step(orc):
    # F3 + SR (Eq.3): over Philox steps, deq(q_H′) − H′ has mean zero (linear step is unbiased)
    gr = inputs.random_graph(16, 30, seed=2)
    heads, hd, F = 2, 4, 8
    H = inputs.features(gr.n, F)
    W, a_src, a_dst = inputs.gat_params(F, heads, hd)
    diffs, smax = [], 0.0
    for step in range(300):
        f = orc.gat_fwd(gr, H, W, a_src, a_dst, heads, hd, bits=8, step=step)
        diffs.append(f["qHp"].astype(np.float64) * f["sHp"][0] - f["Hp"].astype(np.float64))
        smax = max(smax, float(f["sHp"][0]))
    mean = np.mean(diffs, axis=0)
    assert np.max(np.abs(mean)) < 5 * smax / 2 / np.sqrt(300)
    assert np.max(np.abs(diffs)) < smax * (1 + 1e-6)


def test_gcn_quantized_int_aggregation_exact(orc):
    gr = inputs.random_graph(64, 256, seed=3)
    X = inputs.features(gr.n, 20)
    W = inputs.gcn_params(20, 8)
    f = orc.gcn_fwd(gr, X, W, bits=8)
    G = np.zeros((gr.n, gr.n), np.int64)
    G[gr.in_dst(), gr.in_src] = 1
    assert np.array_equal(f["ia"], G @ f["qYs"].astype(np.int64))
    dout = inputs.grad_out(gr.n, 8)
    b = orc.gcn_bwd(gr, f, X, W, dout)
    assert np.array_equal(b["ib"], G.T @ b["qGs"].astype(np.int64))
