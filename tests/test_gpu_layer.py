"""GPU parity of the fused quantized GAT / GCN layers (tango_gat_layer_fwd/bwd,
tango_gcn_layer_fwd/bwd) against the CPU oracle, element by element.

Every int8 tensor, integer accumulator and pinned fp32 value must be bit-exact;
∂a_src / ∂a_dst (the only outputs summed in arbitrary order, with fp32 atomics)
are checked against the recursive-summation error bound derived in DESIGN.md §3:
|err| <= (L + W) * 2^-24 * Σ|terms|, with L + W <= 4096 here.
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


def eq(name, got, want):
    g = got.detach().cpu().numpy() if hasattr(got, "detach") else np.asarray(got)
    w = np.asarray(want)
    assert g.shape == w.shape, f"{name}: shape {g.shape} vs {w.shape}"
    if not np.array_equal(g, w):
        bad = np.argwhere(g != w)
        i = tuple(bad[0])
        raise AssertionError(f"{name}: {len(bad)} / {g.size} differ, first at {i}: {g[i]} vs {w[i]}")


def da_ok(got, want, absum, bound=4096 * 2.0 ** -24):
    g = got.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(g - want) <= bound * absum + 1e-7), np.max(np.abs(g - want) / (absum + 1e-30))


CASES = [
    # name, graph spec, F, heads, head_dim, chunk
    ("toy_like", ("rand", 4, 4, 1), 4, 2, 32, 256),
    ("c0b_h2", ("rand", 64, 256, 0), 16, 2, 32, 256),
    ("c0b_h4", ("rand", 64, 256, 0), 16, 4, 16, 3),
    ("ragged", ("rand", 1000, 4000, 2), 100, 4, 32, 7),
    ("noself", ("noself", 500, 900, 5), 48, 1, 64, 256),
    ("hd512", ("rand", 2000, 20000, 6), 128, 4, 128, 256),
    ("f602", ("rand", 700, 5000, 8), 602, 4, 128, 64),
    # mean in-degree >= 32: the v6 dataflow (gat2.cu) with hub rows (degree > C_E) — split into many
    # canonical chunks at C_E = 7 / 16 / 64 (rows beyond SPIECE chunks fold scratch partials)
    ("v6_h4", ("rand", 800, 30000, 21), 64, 4, 128, 256),
    ("v6_h4_c7", ("rand", 800, 30000, 21), 64, 4, 128, 7),
    ("v6_h2_c64", ("rand", 500, 12000, 22), 32, 2, 64, 64),
    ("v6_h8_c16", ("rand", 400, 10000, 23), 40, 8, 32, 16),
    ("v6_h1", ("rand", 400, 10000, 23), 40, 1, 128, 256),
    ("v6_noself_c64", ("noself", 600, 20000, 24), 48, 4, 64, 64),
]


def build_graph(spec):
    kind, n, d, s = spec
    return inputs.random_graph(n, d, seed=s, self_loops=(kind != "noself"))


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_gat_layer_parity(T, orc, case):
    _gat_parity(T, orc, case, keep_eid=None)


# Without out_eid the source pass recomputes α / ∂α / ∂E_pre from per-node data (the path a
# partitioned graph takes); run it on one GPU by dropping the edge-id map.
@pytest.mark.parametrize("case", [CASES[1], CASES[2], CASES[3], CASES[5]], ids=lambda c: c[0])
def test_gat_layer_parity_recompute_src(T, orc, case):
    _gat_parity(T, orc, case, keep_eid=False)


def _gat_parity(T, orc, case, keep_eid):
    name, spec, F, heads, hd, chunk = case
    gr = build_graph(spec)
    HD = heads * hd
    H = inputs.features(gr.n, F, seed=11)
    W, a_src, a_dst = inputs.gat_params(F, heads, hd, seed=12)
    dH = inputs.grad_out(gr.n, HD, seed=13)
    step, layer_id, slope = 2, 1, 0.2
    dg = T.DeviceGraph(gr, chunk=chunk, keep_eid=keep_eid)
    layer = T.GATLayer(dg, cu(W), cu(a_src), cu(a_dst), heads, hd, slope=slope, bits=8)
    Hout, amax_out = layer.forward(cu(H), step=step, layer_id=layer_id)
    fv = layer.view()
    dHg, dWg, das, dad = layer.backward(cu(dH), step=step, layer_id=layer_id)
    bv = layer.view()
    torch.cuda.synchronize()
    layer.check_status()
    f = orc.gat_fwd(gr, H, W, a_src, a_dst, heads, hd, slope=slope, bits=8, step=step, layer_id=layer_id,
                    chunk=chunk)
    b = orc.gat_bwd(gr, f, H, W, a_src, a_dst, dH)
    # forward: F1-F6
    eq("qH", fv["qH"], f["qH"])
    eq("qW", fv["qW"], f["qW"])
    eq("qWt", fv["qWt"], f["qW"].T)
    eq("scale_H", fv["scalars"][8:9], f["sH"])
    eq("scale_W", fv["scalars"][9:10], f["sW"])
    eq("S", fv["S"], f["S"])
    eq("D", fv["D"], f["Dd"])
    eq("scale_Hp", fv["scalars"][10:11], f["sHp"])
    eq("qHp", fv["qHp"], f["qHp"])
    assert np.all(fv["qHp_full"].cpu().numpy()[:, HD:] == 0)
    eq("qS", fv["qS"], f["qS"])
    eq("qD", fv["qD"], f["qD"])
    eq("m", fv["m"], f["m"])
    eq("den", fv["den"], f["den"])
    if keep_eid is None:
        assert fv["dataflow"] == (2 if name.startswith("v6") else 1), (name, fv["dataflow"])
    if fv["dataflow"] == 1:   # round-1 kernels store α (sign = LeakyReLU branch); v6 recomputes it
        eq("alpha", fv["alpha"], f["alpha"])
        assert np.array_equal(fv["e_pre_pos"].cpu().numpy(), f["e_pre"] > 0)
    eq("H_out", Hout, f["Hout"])
    eq("amax_out", amax_out, f["amax_out"])
    # backward: B1-B9
    eq("qG", bv["qG"], b["qG"])
    if bv["dataflow"] == 1:
        eq("dalpha", bv["dalpha"], b["dalpha"])
        eq("dE_pre", bv["dE_pre"], b["dE_pre"])
    else:   # v6: ∂α in out-CSR order (written by the source pass), ∂E_pre recomputed
        eq("dalpha_out", bv["dalpha_out"], b["dalpha"][gr.out_eid])
    eq("P", bv["P"], b["P"])
    eq("dD", bv["dD"], b["dD"])
    eq("dS", bv["dS"], b["dS"])
    eq("dHp", bv["dHp"], b["dHp"])
    eq("qdHp", bv["qdHp"], b["qdHp"])
    eq("dH", dHg, b["dH"])
    eq("dW", dWg, b["dW"])
    if bv["dataflow"] == 2 or HD % 128 == 0:   # one GPU: the pinned chunk order of R39, bit-exact
        eq("da_src", das, b["da_src"])
        eq("da_dst", dad, b["da_dst"])
    else:
        da_ok(das, b["da_src"], b["da_src_abs"])
        da_ok(dad, b["da_dst"], b["da_dst_abs"])


def test_gat_layer_repeatable_and_hint(T, orc):
    gr = inputs.random_graph(300, 1500, seed=21)
    F, heads, hd = 64, 4, 32
    H = inputs.features(gr.n, F)
    W, a_src, a_dst = inputs.gat_params(F, heads, hd)
    dg = T.DeviceGraph(gr)
    layer = T.GATLayer(dg, cu(W), cu(a_src), cu(a_dst), heads, hd)
    o1, _ = layer.forward(cu(H), step=7)
    o2, _ = layer.forward(cu(H), step=7)
    assert torch.equal(o1, o2)
    hint = cu(np.array([np.abs(H).max()], np.float32))
    o3, _ = layer.forward(cu(H), step=7, amax_hint=hint)
    assert torch.equal(o1, o3)
    o4, _ = layer.forward(cu(H), step=8)
    assert not torch.equal(o1, o4)            # a new Philox step draws new rounding


GCN_CASES = [("c0b", (64, 256, 0), 16, 32), ("cora_like", (2708, 5278, 1), 1433, 128), ("ragged", (999, 3000, 2), 100, 40)]


@pytest.mark.parametrize("case", GCN_CASES, ids=[c[0] for c in GCN_CASES])
def test_gcn_layer_parity(T, orc, case):
    name, (n, d, s), F, O = case
    gr = inputs.random_graph(n, d, seed=s)
    X = inputs.features(gr.n, F, seed=31)
    W = inputs.gcn_params(F, O, seed=32)
    dout = inputs.grad_out(gr.n, O, seed=33)
    dg = T.DeviceGraph(gr)
    layer = T.GCNLayer(dg, cu(W), bits=8)
    out, _ = layer.forward(cu(X), step=1, layer_id=0)
    dX, dW = layer.backward(cu(dout), step=1, layer_id=0)
    v = layer.view()
    torch.cuda.synchronize()
    layer.check_status()
    f = orc.gcn_fwd(gr, X, W, bits=8, step=1, layer_id=0)
    b = orc.gcn_bwd(gr, f, X, W, dout)
    eq("qX", v["qX"], f["qX"])
    eq("qYs", v["qYs"], f["qYs"])
    eq("ia", v["ia"], f["ia"])
    eq("out", out, f["out"])
    eq("qGs", v["qGs"], b["qGs"])
    eq("ib", v["ib"], b["ib"])
    eq("qdY", v["qdY"], b["qdY"])
    eq("dX", dX, b["dX"])
    eq("dW", dW, b["dW"])


def test_layer_validation(T):
    gr = inputs.random_graph(64, 100, seed=1)
    dg = T.DeviceGraph(gr)
    W = torch.zeros((16, 48), device="cuda")
    a = torch.zeros(48, device="cuda")
    with pytest.raises(T.TangoError):        # HD = 48 is not a supported row width
        T.GATLayer(dg, W, a, a, 3, 16)
    W = torch.zeros((16, 64), device="cuda")
    a = torch.zeros(64, device="cuda")
    with pytest.raises(T.TangoError):        # bits outside [2, 8]
        T.GATLayer(dg, W, a, a, 2, 32, bits=1)


def test_v6_variants_subprocess():
    """The v6 alternatives kept behind environment switches (read once per process): P1 scattering ∂α into
    in-CSR order (TANGO_P2_SCATTER), the lane-parallel / multi-segment hub kernels (TANGO_HUB_LANE 1 / 2),
    P2 recomputing α instead of reading F-agg's stored α (TANGO_ALPHA_RECOMPUTE), and P2 gathering ∂α
    instead of reading P1's {∂α, α} records (TANGO_P2_REC=0) — the dense v6 parity cases in a fresh
    process per setting."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for env in ({"TANGO_P2_SCATTER": "1", "TANGO_HUB_LANE": "1"}, {"TANGO_HUB_LANE": "1"}, {"TANGO_P2_SCATTER": "1"},
                {"TANGO_ALPHA_RECOMPUTE": "1"}, {"TANGO_HUB_LANE": "2"}, {"TANGO_HUB_LANE": "2", "TANGO_P2_SCATTER": "1"},
                {"TANGO_HUB_LANE": "2", "TANGO_ALPHA_RECOMPUTE": "1"}, {"TANGO_P2_REC": "0"},
                {"TANGO_P2_REC": "0", "TANGO_HUB_LANE": "2"}, {"TANGO_HUB_P2": "0"}, {"TANGO_HUB_P3": "2"}):
        r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(here, "test_gpu_layer.py"), "-x", "-q",
                            "-k", "v6 and not variants"], env=dict(os.environ, **env), capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, (env, r.stdout[-2000:], r.stderr[-2000:])
