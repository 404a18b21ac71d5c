"""Pins of the oracle's QUANTIZED-mode wiring (reading R8: which operand is int8 at each step; R23:
∂a from the cached deq(q_H′)).

The bypass-mode tests (test_oracle_layer.py) pin the arithmetic of every step against fp64 autograd,
but in quantized mode a shared misreading — aggregating the exact fp32 H′ instead of deq(q_H′),
feeding fp32 S/D into ③, dotting ∂H_out instead of its codes in ⑤″ — would pass those.  Here every
intermediate of the quantized layer is recomputed in float64 with numpy from the oracle's OWN codes
and scales, following the paper's formulas:

  ③  e_pre[e,h] = deq(q_S)[u,h] + deq(q_D)[v,h]                 (S, D int8)
  ④  α = softmax over in-edges of lrelu(e_pre)                   (FP32 per P:604-615)
  ⑤  H_out[v] = Σ_e α[e] · deq(q_H′)[u]
  ⑤″ ∂α[e,h] = s_G s_H′ · Σ_d q_G[v,h,d] q_H′[u,h,d]   (int)
  ④′ P[v] = Σ ∂α α ; ∂E = α(∂α − P[v]) ; ∂E_pre = ∂E·lrelu′
  ③″ ∂D[v] = Σ_{e→v} ∂E_pre ; ③′ ∂S[u] = Σ_{u→v} ∂E_pre
  ⑤′ ∂H′_agg[u] = Σ_{e=(u→v)} α[e] · deq(q_G)[v]
  ②′ ∂H′ = ∂H′_agg + ∂S·a_src + ∂D·a_dst ;  ∂a_src = Σ_u ∂S[u]·deq(q_H′)[u]   (R23)
  ①′ ∂H = deq(q_∂H′ · q_Wᵀ) ; ∂W = deq(q_Hᵀ · q_∂H′)

Each check has a tolerance (fp32 rounding of the oracle's sums, ~1e-6 relative) far below the
difference the corresponding misreading produces (a quantization step, ~1/254 relative); the
`*_discriminates` assertions prove that margin on the same data.
"""
import numpy as np
import pytest

from paper_2308_00890_b200 import inputs


@pytest.fixture(scope="module")
def case(orc):
    gr = inputs.random_graph(96, 500, seed=21)
    heads, hd, F = 4, 16, 24
    H = inputs.features(gr.n, F)
    W, a_src, a_dst = inputs.gat_params(F, heads, hd)
    a_src = a_src * 4.0      # larger attention logits: a non-trivial softmax
    a_dst = a_dst * 4.0
    dH = inputs.grad_out(gr.n, heads * hd)
    slope = 0.2
    f = orc.gat_fwd(gr, H, W, a_src, a_dst, heads, hd, slope=slope, bits=8, chunk=8, step=5)
    b = orc.gat_bwd(gr, f, H, W, a_src, a_dst, dH)
    return dict(gr=gr, heads=heads, hd=hd, F=F, H=H, W=W, a_src=a_src, a_dst=a_dst, dH=dH, slope=slope, f=f, b=b)


def deq(q, s):
    return q.astype(np.float64) * np.float64(s)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def ref_forward(c):
    """float64 recomputation of ③④⑤ from the oracle's codes."""
    gr, f, heads, hd = c["gr"], c["f"], c["heads"], c["hd"]
    src = gr.in_src.astype(np.int64)
    dst = gr.in_dst().astype(np.int64)
    S = deq(f["qS"], f["sS"][0])
    D = deq(f["qD"], f["sD"][0])
    e_pre = S[src] + D[dst]
    el = np.where(e_pre > 0, e_pre, e_pre * c["slope"])
    m = np.full((gr.n, heads), -np.inf)
    np.maximum.at(m, dst, el)
    ex = np.exp(el - m[dst])
    den = np.zeros((gr.n, heads))
    np.add.at(den, dst, ex)
    alpha = ex / den[dst]
    Hp = deq(f["qHp"], f["sHp"][0]).reshape(gr.n, heads, hd)
    Hout = np.zeros((gr.n, heads, hd))
    np.add.at(Hout, dst, alpha[:, :, None] * Hp[src])
    return dict(e_pre=e_pre, alpha=alpha, Hout=Hout.reshape(gr.n, heads * hd), src=src, dst=dst)


def test_sddmm_add_uses_quantized_S_D(case):
    f = case["f"]
    r = ref_forward(case)
    assert rel(f["e_pre"], r["e_pre"]) < 1e-6
    # misreading: fp32 S and D fed into ③
    wrong = f["S"].astype(np.float64)[r["src"]] + f["Dd"].astype(np.float64)[r["dst"]]
    assert rel(wrong, r["e_pre"]) > 100 * 1e-6


def test_softmax_of_quantized_logits(case):
    f = case["f"]
    r = ref_forward(case)
    assert np.max(np.abs(f["alpha"] - r["alpha"])) < 2e-6


def test_spmm_aggregates_dequantized_codes(case):
    f = case["f"]
    r = ref_forward(case)
    assert rel(f["Hout"], r["Hout"]) < 2e-6
    # misreading: the exact fp32 H′ aggregated instead of deq(q_H′)
    gr, heads, hd = case["gr"], case["heads"], case["hd"]
    Hp = f["Hp"].astype(np.float64).reshape(gr.n, heads, hd)
    wrong = np.zeros((gr.n, heads, hd))
    np.add.at(wrong, r["dst"], r["alpha"][:, :, None] * Hp[r["src"]])
    assert rel(wrong.reshape(gr.n, -1), r["Hout"]) > 100 * 2e-6
    assert f["amax_out"][0] == np.abs(f["Hout"]).max()


def test_backward_wiring(case):
    gr, f, b, heads, hd = case["gr"], case["f"], case["b"], case["heads"], case["hd"]
    r = ref_forward(case)
    src, dst = r["src"], r["dst"]
    n = gr.n
    # ⑤″ on codes: exact integers times the fp32 product of the two scales
    qG = b["qG"].astype(np.int64).reshape(n, heads, hd)
    qHp = f["qHp"].astype(np.int64).reshape(n, heads, hd)
    idot = np.einsum("ehd,ehd->eh", qG[dst], qHp[src])
    sGH = np.float32(b["sG"][0]) * np.float32(f["sHp"][0])
    assert np.array_equal(b["dalpha"], idot.astype(np.float32) * sGH)
    # misreading: fp32 ∂H_out dotted with deq(q_H′)
    dHf = case["dH"].astype(np.float64).reshape(n, heads, hd)
    wrong = np.einsum("ehd,ehd->eh", dHf[dst], deq(f["qHp"], f["sHp"][0]).reshape(n, heads, hd)[src])
    assert rel(wrong, b["dalpha"]) > 1e-4
    # ④′ from the oracle's α and ∂α
    al = f["alpha"].astype(np.float64)
    da = b["dalpha"].astype(np.float64)
    P = np.zeros((n, heads))
    np.add.at(P, dst, da * al)
    assert np.max(np.abs(b["P"] - P)) <= 1e-6 * max(1.0, np.abs(P).max())
    dE = al * (da - P[dst])
    ep = f["e_pre"].astype(np.float64)
    dEp = np.where(ep > 0, dE, dE * case["slope"])
    sc = np.abs(dEp).max()
    assert np.max(np.abs(b["dE_pre"] - dEp)) <= 1e-5 * sc
    # ③″ / ③′ incidence sums
    dD = np.zeros((n, heads))
    np.add.at(dD, dst, dEp)
    dS = np.zeros((n, heads))
    np.add.at(dS, src, dEp)
    assert np.max(np.abs(b["dD"] - dD)) <= 1e-5 * sc * 4
    assert np.max(np.abs(b["dS"] - dS)) <= 1e-5 * sc * 4
    # ⑤′ aggregates deq(q_G) over out-edges with the forward's α
    G = deq(b["qG"], b["sG"][0]).reshape(n, heads, hd)
    agg = np.zeros((n, heads, hd))
    np.add.at(agg, src, al[:, :, None] * G[dst])
    agg = agg.reshape(n, -1)
    assert rel(b["dHp_agg"], agg) < 2e-6
    wrong = np.zeros((n, heads, hd))
    np.add.at(wrong, src, al[:, :, None] * dHf[dst])
    assert rel(wrong.reshape(n, -1), agg) > 100 * 2e-6
    # ②′ chain rule; ∂a from the cached deq(q_H′) (R23), not from the fp32 H′
    a_s = case["a_src"].astype(np.float64).reshape(heads, hd)
    a_d = case["a_dst"].astype(np.float64).reshape(heads, hd)
    dS_o = b["dS"].astype(np.float64)
    dD_o = b["dD"].astype(np.float64)
    dHp = (b["dHp_agg"].astype(np.float64).reshape(n, heads, hd) + dS_o[:, :, None] * a_s[None]
           + dD_o[:, :, None] * a_d[None]).reshape(n, -1)
    assert rel(b["dHp"], dHp) < 2e-6
    Hq = deq(f["qHp"], f["sHp"][0]).reshape(n, heads, hd)
    da_src = np.einsum("nh,nhd->hd", dS_o, Hq).reshape(-1)
    da_dst = np.einsum("nh,nhd->hd", dD_o, Hq).reshape(-1)
    assert np.all(np.abs(b["da_src"] - da_src) <= 1e-5 * b["da_src_abs"] + 1e-12)
    assert np.all(np.abs(b["da_dst"] - da_dst) <= 1e-5 * b["da_dst_abs"] + 1e-12)
    Hf = f["Hp"].astype(np.float64).reshape(n, heads, hd)
    wrong = np.einsum("nh,nhd->hd", dS_o, Hf).reshape(-1)
    assert np.max(np.abs(wrong - da_src) / (b["da_src_abs"] + 1e-30)) > 10 * 1e-5
    # B8: q_∂H′ are SR codes of ∂H′ (within one step), ①′ from the cached q_H / q_W
    assert np.max(np.abs(deq(b["qdHp"], b["sdHp"][0]) - b["dHp"])) < b["sdHp"][0] * (1 + 1e-6)
    acc = b["qdHp"].astype(np.int64) @ f["qW"].astype(np.int64).T
    assert np.array_equal(b["dH"], acc.astype(np.float32) * (np.float32(b["sdHp"][0]) * np.float32(f["sW"][0])))
    accw = f["qH"].astype(np.int64).T @ b["qdHp"].astype(np.int64)
    assert np.array_equal(b["dW"], accw.astype(np.float32) * (np.float32(f["sH"][0]) * np.float32(b["sdHp"][0])))


def test_forward_quantizer_inputs(case):
    """F1/F3/F4: q_H, q_H′, q_S, q_D are SR codes of H, H′ = deq(q_H·q_W), S and D from the exact fp32 H′
    (R10), each within one quantization step."""
    f, c = case["f"], case
    heads, hd = c["heads"], c["hd"]
    assert np.max(np.abs(deq(f["qH"], f["sH"][0]) - c["H"])) < f["sH"][0] * (1 + 1e-6)
    acc = f["qH"].astype(np.int64) @ f["qW"].astype(np.int64)
    Hp = acc.astype(np.float32) * (np.float32(f["sH"][0]) * np.float32(f["sW"][0]))
    assert np.array_equal(f["Hp"], Hp)
    assert np.max(np.abs(deq(f["qHp"], f["sHp"][0]) - Hp)) < f["sHp"][0] * (1 + 1e-6)
    n = Hp.shape[0]
    S = np.einsum("nhd,hd->nh", Hp.astype(np.float64).reshape(n, heads, hd), c["a_src"].reshape(heads, hd))
    D = np.einsum("nhd,hd->nh", Hp.astype(np.float64).reshape(n, heads, hd), c["a_dst"].reshape(heads, hd))
    assert rel(f["S"], S) < 1e-5 and rel(f["Dd"], D) < 1e-5
    assert np.max(np.abs(deq(f["qS"], f["sS"][0]) - f["S"])) < f["sS"][0] * (1 + 1e-6)
    assert np.max(np.abs(deq(f["qD"], f["sD"][0]) - f["Dd"])) < f["sD"][0] * (1 + 1e-6)
