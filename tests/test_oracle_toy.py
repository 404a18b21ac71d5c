"""The paper's worked two-head toy example (§2.1, Fig.1) fed step by step
through the oracle's primitives (bypass mode = the paper's full-precision
illustration).  Expected values come from tests/golden/toy_gat.json, each cited.
"""
import json
import os

import numpy as np
import pytest

from paper_2308_00890_b200 import inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "toy_gat.json")))
TOL = GOLD["tolerance"]


def g(key):
    return np.array(GOLD[key]["value"], np.float64)


@pytest.fixture(scope="module")
def toy():
    gr = inputs.toy_graph()
    # edge ids are in-CSR positions and equal the paper's e0..e4
    src = gr.in_src.tolist()
    dst = gr.in_dst().tolist()
    assert list(zip(src, dst)) == [tuple(x) for x in GOLD["edges_src_dst"]]
    return gr


def test_step2_projection(orc, toy):
    # ② S = (H'·a_src)ᵀ per head, via the layer in bypass mode with W = I so that H' = H exactly.
    H = np.zeros((4, 4), np.float32)
    H[0] = g("Hp_v0")
    H[1] = g("Hp_v1")
    W = np.eye(4, dtype=np.float32)
    a_src = g("a_src").astype(np.float32)
    a_dst = np.zeros(4, np.float32)
    f = orc.gat_fwd(toy, H, W, a_src, a_dst, heads=2, head_dim=2, slope=0.0, bits=0)
    assert np.array_equal(f["Hp"][0], H[0])
    assert np.allclose(f["S"][0], g("S_v0"), atol=TOL)


def test_step3_sddmm_add_leakyrelu(orc, toy):
    S = np.zeros((4, 2), np.float32)
    D = np.zeros((4, 2), np.float32)
    S[0] = g("S_v0")
    D[3] = g("D_v3")
    e_pre, el = orc.sddmm_add(toy, 2, orc.qref(v=S), orc.qref(v=D), 0.0)
    assert np.allclose(e_pre[3], g("E_pre_e3"), atol=TOL)
    assert np.allclose(el[3], g("E_e3"), atol=TOL)
    assert el[3, 1] == 0.0


def test_step4_edge_softmax(orc, toy):
    el = np.zeros((5, 2), np.float32)
    el[3] = g("E_e3")
    el[4] = g("E_e4")
    el[0] = [0.3, -2.0]
    el[1] = [5.0, 1.0]
    el[2] = [-1.0, 0.0]
    m, den, alpha = orc.edge_softmax(toy, 2, el)
    assert np.allclose(alpha[3], g("alpha_e3"), atol=TOL)
    assert np.allclose(alpha[4], g("alpha_e4"), atol=TOL)
    # single in-edge => alpha == 1 exactly ("1.0x")
    assert np.all(alpha[:3] == 1.0)


def test_step5p_spmm_reversed(orc, toy):
    # ⑤′ ∂H′ = (Gᵀ⊙α)·∂H_out; ∂H′[v1] gathers e0 (to v0) and e2 (to v2), α = 1
    dH = np.zeros((4, 4), np.float32)
    dH[0] = g("dHout_v0")
    dH[2] = g("dHout_v2")
    alpha = np.ones((5, 2), np.float32)
    out = orc.spmm_alpha(toy, 1, 2, 4, alpha, orc.qref(v=dH))
    assert np.allclose(out[1], g("dHp_agg_v1"), atol=TOL)


def test_step5pp_sddmm_dot(orc, toy):
    # ⑤″ ∂α[e0] = ∂H_out[v0] · H′[v1] per head
    dH = np.zeros((4, 4), np.float32)
    dH[0] = g("dHout_v0")
    Hp = np.zeros((4, 4), np.float32)
    Hp[1] = g("Hp_v1")
    da = orc.sddmm_dot(toy, 2, 4, orc.qref(v=dH), orc.qref(v=Hp))
    assert np.allclose(da[0], g("dalpha_e0"), atol=TOL)


def _v3_backward(orc, toy):
    el = np.zeros((5, 2), np.float32)
    el[3] = g("E_e3")
    el[4] = g("E_e4")
    e_pre = el.copy()
    e_pre[3] = g("E_pre_e3")
    _, _, alpha = orc.edge_softmax(toy, 2, el)
    dalpha = np.zeros((5, 2), np.float32)
    dalpha[3, 0] = g("dalpha_e3_h0")
    dalpha[4, 0] = g("dalpha_e4_h0")
    dalpha[3, 1] = 0.0      # head-1 values not printed; difference 0.60 (Appendix A)
    dalpha[4, 1] = 0.60
    dalpha[0] = [0.78, -0.13]
    P, dE, dEp = orc.softmax_bwd(toy, 2, alpha, dalpha, e_pre, 0.0)
    return alpha, dalpha, P, dE, dEp


def test_step4p_softmax_backward(orc, toy):
    alpha, dalpha, P, dE, dEp = _v3_backward(orc, toy)
    assert abs(P[3, 0] - g("P_v3_h0")) < TOL
    assert abs(dE[3, 0] - g("dE_e3_h0")) < TOL
    # single in-edge => ∂E == 0 exactly (P = fma(∂α, 1, 0) = ∂α)
    assert np.all(dE[:3] == 0.0)


def test_step3p_incidence_spmm(orc, toy):
    alpha, dalpha, P, dE, dEp = _v3_backward(orc, toy)
    dD = orc.edge_sum(toy, 0, 2, dEp)
    dS = orc.edge_sum(toy, 1, 2, dEp)
    assert np.allclose(dD[3], g("dD_v3"), atol=TOL)
    assert np.allclose(dS[3], g("dS_v3"), atol=TOL)
    # head 0 of v3: softmax gradients over the in-edges sum to zero (both e_pre > 0)
    assert abs(dD[3, 0]) < 1e-6
