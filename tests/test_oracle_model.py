"""Pins of the NEXT-1 oracle functions: the full-precision GEMM order (R33), the
full-precision final GAT layer (R35), bias + ReLU (R34), cross-entropy (R36), the FP32
master-weight update (Eq.5-6) and the composed multi-layer training step.

Every pin is against something other than the oracle itself: exact integer arithmetic, a closed
form that only the chunked order produces, fp64 numpy / torch autograd of the textbook model.
"""
import math

import numpy as np
import pytest
import torch

from paper_2308_00890_b200 import inputs
from test_oracle_layer import torch_gat


def _ints(shape, seed, lo=-8, hi=9):
    return np.random.Generator(np.random.PCG64(seed)).integers(lo, hi, size=shape).astype(np.float32)


@pytest.mark.parametrize("tA,tB", [(False, False), (True, False), (False, True), (True, True)])
def test_sgemm_exact_on_integers(orc, tA, tB):
    # |partial sums| < 2^24: every fp32 op is exact, so any order gives the integer product;
    # a transposed operand or a wrong index changes the values.  K = 3000 spans 3 chunks.
    M, N, K = 37, 29, 3000
    A, B = _ints((M, K), 1), _ints((K, N), 2)
    want = A.astype(np.int64) @ B.astype(np.int64)
    got = orc.sgemm(A.T.copy() if tA else A, B.T.copy() if tB else B, transA=tA, transB=tB)
    assert np.array_equal(got.astype(np.int64), want)


def test_sgemm_chunk_order_closed_form(orc):
    # R33: chunks of 1024 k, partials folded left to right.  Terms: 2^24 then 2047 ones.
    # Chunk 0 = 2^24 (each +1 rounds back to 2^24, ties to even); chunk 1 = 1024 exactly;
    # total = 2^24 + 1024.  A plain sequential chain would give 2^24, one chunk per k 2^24 + 2047.
    K = 2048
    A = np.ones((1, K), np.float32)
    B = np.ones((K, 1), np.float32)
    B[0, 0] = 2.0 ** 24
    assert orc.sgemm(A, B)[0, 0] == np.float32(2.0 ** 24 + 1024)
    x = np.ones((K, 1), np.float32)
    x[0, 0] = 2.0 ** 24
    assert orc.colsum(x)[0] == np.float32(2.0 ** 24 + 1024)


def test_sgemm_vs_fp64(orc):
    rng = np.random.Generator(np.random.PCG64(3))
    A = rng.standard_normal((50, 2500)).astype(np.float32)
    B = rng.standard_normal((2500, 40)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    bound = (1024 + 3) * 2.0 ** -24 * (np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64))
    assert np.all(np.abs(orc.sgemm(A, B) - ref) <= bound)


def test_bias_relu(orc):
    rng = np.random.Generator(np.random.PCG64(4))
    x = rng.standard_normal((300, 24)).astype(np.float32)
    b = rng.standard_normal(24).astype(np.float32)
    a, am = orc.bias_relu_fwd(x, b)
    y = (x.astype(np.float64) + b).astype(np.float32)       # one rn add, exact in fp64 first
    assert np.array_equal(a, np.maximum(y, 0))
    assert am == a.max()
    da = rng.standard_normal((300, 24)).astype(np.float32)
    dx, db, amd = orc.bias_relu_bwd(a, da)
    assert np.array_equal(dx, np.where(y > 0, da, 0).astype(np.float32))
    assert amd == np.abs(dx).max()
    ref = dx.astype(np.float64).sum(0)
    assert np.all(np.abs(db - ref) <= 310 * 2.0 ** -24 * np.abs(dx).astype(np.float64).sum(0))


def test_cross_entropy_closed_forms(orc):
    n, C = 10, 7
    lab = np.arange(n, dtype=np.int32) % C
    lab[3] = -1
    loss, dz, rl = orc.cross_entropy(np.full((n, C), 0.37, np.float32), lab)
    assert abs(loss - math.log(C)) < 1e-6                      # uniform logits: ln C
    onehot = np.zeros((n, C))
    onehot[np.arange(n), np.maximum(lab, 0)] = 1
    want = (1.0 / C - onehot) / 9
    want[3] = 0
    assert np.allclose(dz, want, atol=1e-7)
    assert np.all(dz[3] == 0) and rl[3] == 0
    z = np.zeros((2, 3), np.float32)
    z[0, 1] = z[1, 2] = 80.0                                   # correct class dominant: loss -> 0
    loss, dz, _ = orc.cross_entropy(z, np.array([1, 2], np.int32))
    assert loss < 1e-30 and np.abs(dz).max() < 1e-30
    with pytest.raises(orc.OracleError):
        orc.cross_entropy(z, np.array([1, 3], np.int32))


def test_cross_entropy_vs_torch(orc):
    rng = np.random.Generator(np.random.PCG64(6))
    z = (rng.standard_normal((200, 40)) * 3).astype(np.float32)
    lab = inputs.labels(200, 40, train_frac=0.6, seed=7)
    loss, dz, _ = orc.cross_entropy(z, lab)
    zt = torch.tensor(z, dtype=torch.float64, requires_grad=True)
    lt = torch.from_numpy(lab.astype(np.int64))
    ref = torch.nn.functional.cross_entropy(zt, lt, ignore_index=-1)
    ref.backward()
    assert abs(loss - ref.item()) < 1e-5 * abs(ref.item())
    assert np.abs(dz - zt.grad.numpy()).max() < 1e-8


def test_sgd_update(orc):
    rng = np.random.Generator(np.random.PCG64(8))
    w = rng.standard_normal(1000).astype(np.float32)
    g = rng.standard_normal(1000).astype(np.float32)
    assert np.array_equal(orc.sgd(w, g, 0.0), w)
    got = orc.sgd(w, g, 0.01)
    ref = w.astype(np.float64) - np.float64(np.float32(0.01)) * g.astype(np.float64)
    assert np.all(np.abs(got - ref) <= 2.0 ** -23 * (np.abs(ref) + np.abs(w)))


def test_add_then_quantize_retains_small_updates(orc):
    # Eq.5 vs Eq.6: 100 updates of 0.004 < s/2 (grid s = 0.1 after the master is
    # quantized with nearest rounding).  Quantize-then-add (Q(W)+Q(ΔW)) never moves; the FP32
    # master (add, then quantize at use) accumulates 0.4 and its quantization moves 4 steps.
    s = np.float32(0.1)
    q = lambda x: np.float32(np.rint(x / s) * s)
    w_q = q(np.float32(0.26))
    master = np.array([0.26], np.float32)
    for _ in range(100):
        w_q = q(w_q + q(np.float32(0.004)))                    # Eq.5
        master = orc.sgd(master, np.array([-0.004], np.float32), 1.0)   # W − lr·∂W with ∂W = −ΔW
    assert w_q == q(np.float32(0.26))
    assert abs(master[0] - 0.66) < 1e-5 and q(master[0]) == np.float32(0.7)


def torch_gat_out(gr, H, W, a_src, a_dst, b, heads, C, slope):
    out, _ = torch_gat(gr, H, W, a_src, a_dst, heads, C, slope)
    return out.view(gr.n, heads, C).mean(1) + b


@pytest.mark.parametrize("n,draws,heads,C,F,seed", [(40, 100, 2, 5, 16, 1), (64, 256, 4, 7, 24, 2),
                                                    (30, 60, 1, 3, 9, 3)])
def test_gat_out_layer_vs_autograd(orc, n, draws, heads, C, F, seed):
    gr = inputs.random_graph(n, draws, seed=seed)
    H = inputs.features(gr.n, F, seed=seed + 1)
    W, a_src, a_dst = inputs.gat_params(F, heads, C, seed=seed + 2)
    bias = inputs.features(1, C, seed=seed + 4)[0]
    dz = inputs.grad_out(gr.n, C, seed=seed + 3)
    f = orc.gat_out_fwd(gr, H, W, a_src, a_dst, bias, heads, C, slope=0.2, chunk=3)
    bo = orc.gat_out_bwd(gr, f, H, W, a_src, a_dst, dz)
    T = lambda a: torch.tensor(a, dtype=torch.float64, requires_grad=True)
    Ht, Wt, ast, adt, bt = T(H), T(W), T(a_src), T(a_dst), T(bias)
    z = torch_gat_out(gr, Ht, Wt, ast, adt, bt, heads, C, 0.2)
    z.backward(torch.tensor(dz, dtype=torch.float64))
    rel = lambda a, b: np.linalg.norm(np.asarray(a, np.float64) - b.detach().numpy()) / max(
        np.linalg.norm(b.detach().numpy()), 1e-3)
    assert rel(f["logits"], z) < 1e-5
    for got, ref in [(bo["dH"], Ht.grad), (bo["dW"], Wt.grad), (bo["da_src"], ast.grad), (bo["da_dst"], adt.grad),
                     (bo["db"], bt.grad)]:
        assert rel(got, ref) < 1e-5


def _torch_model_loss(gr, X, hidden, out, labels, slope):
    T = lambda a: torch.tensor(a, dtype=torch.float64, requires_grad=True)
    leaves = []
    h = torch.tensor(X, dtype=torch.float64)
    for p in hidden:
        ps = {k: T(p[k]) for k in ("W", "a_src", "a_dst", "b")}
        leaves.append(ps)
        o, _ = torch_gat(gr, h, ps["W"], ps["a_src"], ps["a_dst"], p["heads"], p["head_dim"], slope)
        h = torch.relu(o + ps["b"])
    ps = {k: T(out[k]) for k in ("W", "a_src", "a_dst", "b")}
    leaves.append(ps)
    z = torch_gat_out(gr, h, ps["W"], ps["a_src"], ps["a_dst"], ps["b"], out["heads"], out["classes"], slope)
    loss = torch.nn.functional.cross_entropy(z, torch.from_numpy(labels.astype(np.int64)), ignore_index=-1)
    loss.backward()
    return loss.item(), leaves


@pytest.mark.parametrize("layers,seed", [(2, 11), (3, 12)])
def test_model_step_bypass_vs_autograd(orc, layers, seed):
    # bits = 0 turns quantization off: the composed step (layer order, bias/ReLU wiring, head mean,
    # loss, every gradient) must equal fp64 autograd of the textbook model to fp32 rounding.
    gr = inputs.random_graph(48, 150, seed=seed)
    X = inputs.features(gr.n, 12, seed=seed + 1)
    hidden, out = inputs.gat_model_params(12, 2, 6, layers, 5, bias_scale=0.3, seed=seed + 2)
    lab = inputs.labels(gr.n, 5, train_frac=0.7, seed=seed + 3)
    r = orc.gat_model_step(gr, X, hidden, out, lab, lr=0.5, bits=0, chunk=4)
    loss, leaves = _torch_model_loss(gr, X, hidden, out, lab, 0.2)
    assert abs(r["loss"] - loss) < 1e-5 * abs(loss)
    grads = r["grads"] + [r["out_grads"]]
    for gr_o, lv in zip(grads, leaves):
        for k in ("W", "a_src", "a_dst", "b"):
            ref = lv[k].grad.numpy()
            assert np.linalg.norm(gr_o[k] - ref) <= 1e-5 * max(np.linalg.norm(ref), 1e-6), k
    # the update is W − lr·∂W on every FP32 master
    for p_new, p_old, gr_o in zip(r["hidden"] + [r["out"]], hidden + [out], grads):
        for k in ("W", "a_src", "a_dst", "b"):
            assert np.allclose(p_new[k], p_old[k] - 0.5 * gr_o[k], rtol=1e-6, atol=1e-7)


def test_model_step_quantized_trains(orc):
    # Quantized hidden layer (int8 SR) + FP32 final layer: the step is reproducible bit for bit under
    # the same Philox step; full-batch SGD lowers the loss, and the quantized trajectory tracks the
    # unquantized one (the paper's accuracy claim, at toy scale).
    gr = inputs.random_graph(64, 256, seed=21)
    X = inputs.features(gr.n, 16, seed=22)
    lab = inputs.labels(gr.n, 4, seed=25)
    hidden0, out0 = inputs.gat_model_params(16, 4, 8, 2, 4, seed=23)
    r1 = orc.gat_model_step(gr, X, hidden0, out0, lab, lr=0.0, bits=8, step=5)
    r2 = orc.gat_model_step(gr, X, hidden0, out0, lab, lr=0.0, bits=8, step=5)
    assert r1["loss"] == r2["loss"] and np.array_equal(r1["out_grads"]["W"], r2["out_grads"]["W"])
    final = {}
    for bits in (0, 8):
        hidden, out = hidden0, out0
        losses = []
        for it in range(30):
            r = orc.gat_model_step(gr, X, hidden, out, lab, lr=1.0, bits=bits, step=it)
            losses.append(r["loss"])
            hidden, out = r["hidden"], r["out"]
        assert losses[-1] < 0.9 * losses[0], losses
        final[bits] = losses[-1]
    assert abs(final[8] - final[0]) < 0.02 * final[0], final


def torch_gcn_bias(gr, X, W, b):
    from test_oracle_layer import torch_gcn
    return torch_gcn(gr, X, W) + b


def test_gather_sum_dense(orc):
    # unweighted chunked gather = dense adjacency products (in: A·x, out: Aᵀ·x) within fp32 rounding
    gr = inputs.random_graph(60, 300, seed=31)
    x = inputs.features(gr.n, 5, seed=32)
    A = np.zeros((gr.n, gr.n))
    A[gr.in_dst(), gr.in_src] = 1.0
    for d, M in ((0, A), (1, A.T)):
        got = orc.gather_sum(gr, d, x, chunk=3)
        ref = M @ x.astype(np.float64)
        assert np.all(np.abs(got - ref) <= 64 * 2.0 ** -24 * (np.abs(M) @ np.abs(x.astype(np.float64))))


@pytest.mark.parametrize("layers,seed", [(2, 41), (3, 42)])
def test_gcn_model_step_bypass_vs_autograd(orc, layers, seed):
    gr = inputs.random_graph(50, 160, seed=seed)
    X = inputs.features(gr.n, 20, seed=seed + 1)
    hidden, out = inputs.gcn_model_params(20, 16, layers, 4, bias_scale=0.3, seed=seed + 2)
    lab = inputs.labels(gr.n, 4, train_frac=0.7, seed=seed + 3)
    r = orc.gcn_model_step(gr, X, hidden, out, lab, lr=0.5, bits=0, chunk=4)
    T = lambda a: torch.tensor(a, dtype=torch.float64, requires_grad=True)
    h = torch.tensor(X, dtype=torch.float64)
    leaves = []
    for p in hidden:
        ps = {k: T(p[k]) for k in ("W", "b")}
        leaves.append(ps)
        h = torch.relu(torch_gcn_bias(gr, h, ps["W"], ps["b"]))
    ps = {k: T(out[k]) for k in ("W", "b")}
    leaves.append(ps)
    z = torch_gcn_bias(gr, h, ps["W"], ps["b"])
    loss = torch.nn.functional.cross_entropy(z, torch.from_numpy(lab.astype(np.int64)), ignore_index=-1)
    loss.backward()
    assert abs(r["loss"] - loss.item()) < 1e-5 * abs(loss.item())
    assert np.linalg.norm(r["logits"] - z.detach().numpy()) < 1e-5 * np.linalg.norm(z.detach().numpy())
    for gr_o, lv in zip(r["grads"] + [r["out_grads"]], leaves):
        for k in ("W", "b"):
            ref = lv[k].grad.numpy()
            assert np.linalg.norm(gr_o[k] - ref) <= 1e-5 * max(np.linalg.norm(ref), 1e-6), k
