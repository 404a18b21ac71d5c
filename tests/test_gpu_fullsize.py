"""Full-size parity: the arxiv-shaped GAT layer exactly as bench.py times it (BASELINE.json
configs[2]: N = 169,343, E = 2.27 M after augmentation, F = 128, 4 heads x 128, C_E = 256, one GPU,
the same seeded inputs), checked against the full CPU oracle on every output element.

Every int8 tensor, integer accumulator and fp32 output is compared bit for bit; ∂a_src / ∂a_dst
within the recursive-summation bound of DESIGN.md §3.  The oracle takes a few seconds on the GPU
box's host cores (OpenMP rows, bit-identical to one thread).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from paper_2308_00890_b200 import inputs  # noqa: E402


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_00890_b200 import tango
    tango.load()
    return tango


def eq(name, got, want):
    g = got.detach().cpu().numpy() if hasattr(got, "detach") else np.asarray(got)
    w = np.asarray(want)
    assert g.shape == w.shape, f"{name}: shape {g.shape} vs {w.shape}"
    if not np.array_equal(g, w):
        bad = np.argwhere(g != w)
        i = tuple(bad[0])
        raise AssertionError(f"{name}: {len(bad)} / {g.size} differ, first at {i}: {g[i]} vs {w[i]}")


def test_gat_layer_arxiv_full_size(T, orc):
    kw, F, H, D = inputs.WORKLOADS["arxiv"]
    g = inputs.workload_graph("arxiv")
    HD = H * D
    W, a_s, a_d = inputs.gat_params(F, H, D)
    X = inputs.features(g.n, F)
    dY = inputs.grad_out(g.n, HD)
    step, layer_id = 7, 0
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    dg = T.DeviceGraph(g)                      # chunk_edges 256, out_eid present (one GPU)
    layer = T.GATLayer(dg, cu(W), cu(a_s), cu(a_d), H, D, slope=0.2, bits=8)
    Hout, amax_out = layer.forward(cu(X), step=step, layer_id=layer_id)
    fv = layer.view()
    dX, dW, das, dad = layer.backward(cu(dY), step=step, layer_id=layer_id)
    bv = layer.view()
    torch.cuda.synchronize()
    layer.check_status()

    f = orc.gat_fwd(g, X, W, a_s, a_d, H, D, slope=0.2, bits=8, step=step, layer_id=layer_id, chunk=256)
    b = orc.gat_bwd(g, f, X, W, a_s, a_d, dY)
    eq("qH", fv["qH"], f["qH"])
    eq("qHp", fv["qHp"], f["qHp"])
    eq("S", fv["S"], f["S"])
    eq("D", fv["D"], f["Dd"])
    eq("m", fv["m"], f["m"])
    eq("den", fv["den"], f["den"])
    if fv["dataflow"] == 1:
        eq("alpha", fv["alpha"], f["alpha"])
    eq("H_out", Hout, f["Hout"])
    eq("amax_out", amax_out, f["amax_out"])
    eq("qG", bv["qG"], b["qG"])
    if bv["dataflow"] == 1:
        eq("dalpha", bv["dalpha"], b["dalpha"])
        eq("dE_pre", bv["dE_pre"], b["dE_pre"])
    else:
        eq("dalpha_out", bv["dalpha_out"], b["dalpha"][g.out_eid])
        eq("dS", bv["dS"], b["dS"])
    eq("P", bv["P"], b["P"])
    eq("dD", bv["dD"], b["dD"])
    eq("dHp", bv["dHp"], b["dHp"])
    eq("qdHp", bv["qdHp"], b["qdHp"])
    eq("dH", dX, b["dH"])
    eq("dW", dW, b["dW"])
    if True:   # one GPU, HD = 512: the pinned chunk order of R39 on either dataflow, bit-exact
        eq("da_src", das, b["da_src"])
        eq("da_dst", dad, b["da_dst"])
    else:
        bound = 4096 * 2.0 ** -24
        for name, got, want, absum in (("da_src", das, b["da_src"], b["da_src_abs"]),
                                       ("da_dst", dad, b["da_dst"], b["da_dst_abs"])):
            err = np.abs(got.cpu().numpy().astype(np.float64) - want)
            assert np.all(err <= bound * absum + 1e-7), (name, float(np.max(err / (absum + 1e-30))))
    # the hub rows (max in-degree ~8K, > 31 canonical chunks) are inside this comparison
    assert int(np.diff(g.in_ptr).max()) > 30 * 256


def test_gat_train_step_arxiv_full_size(T, orc):
    """NEXT-1 at full size: one training step of the 3-layer arxiv GAT exactly as bench.py's train_step
    builds it (same seeded graph, features, parameters, labels, lr), against oracle.gat_model_step."""
    from paper_2308_00890_b200.model import GATModel
    from test_gpu_layer import da_ok
    kw, F, H, D = inputs.WORKLOADS["arxiv"]
    g = inputs.workload_graph("arxiv")
    C = inputs.ARXIV_CLASSES
    hidden, out = inputs.gat_model_params(F, H, D, 3, C)
    X = inputs.features(g.n, F)
    lab = inputs.labels(g.n, C, train_frac=inputs.ARXIV_TRAIN_FRAC)
    n_lab = int((lab >= 0).sum())
    lr, step = 0.01, 2
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    dev = lambda p: {k: (cu(v) if isinstance(v, np.ndarray) else v) for k, v in p.items()}
    hid_d, out_d = [dev(p) for p in hidden], dev(out)
    model = GATModel(T.DeviceGraph(g), hid_d, out_d, slope=0.2, bits=8)
    loss = model.step(cu(X), cu(lab), n_lab, lr, step=step)
    torch.cuda.synchronize()
    model.check_status()
    r = orc.gat_model_step(g, X, hidden, out, lab, lr=lr, bits=8, step=step, chunk=256)
    assert abs(loss.item() - r["loss"]) <= 1e-6 * abs(r["loss"])
    eq("logits", model.logits, r["logits"])
    for l in range(2):
        eq(f"act{l}", model.act[l], r["hs"][l + 1])
        eq(f"dW{l}", model.grads[l]["W"], r["grads"][l]["W"])
        eq(f"db{l}", model.grads[l]["b"], r["grads"][l]["b"])
        da_ok(model.grads[l]["a_src"], r["grads"][l]["a_src"], r["grads"][l]["da_src_abs"])
        eq(f"W{l} updated", hid_d[l]["W"], r["hidden"][l]["W"])
    og = r["out_grads"]
    eq("out dW", model.out_grads["W"], og["W"])
    eq("out db", model.out_grads["b"], og["b"])
    da_ok(model.out_grads["a_src"], og["a_src"], og["da_src_abs"])
    da_ok(model.out_grads["a_dst"], og["a_dst"], og["da_dst_abs"])
    eq("out W updated", out_d["W"], r["out"]["W"])


@pytest.mark.skipif(not __import__("os").environ.get("TANGO_FULL_PRODUCTS"),
                    reason="set TANGO_FULL_PRODUCTS=1 (about 10 min: graph build + oracle on 123 M edges)")
def test_gat_layer_products_full_size(T, orc):
    """BASELINE.json configs[4] on one GPU (products-shaped: N = 2.45 M, E = 123 M, F = 100, 4 x 128,
    tables 10x the L2): every output of the layer against the full oracle."""
    kw, F, H, D = inputs.WORKLOADS["products"]
    g = inputs.workload_graph("products")
    W, a_s, a_d = inputs.gat_params(F, H, D)
    X = inputs.features(g.n, F)
    dY = inputs.grad_out(g.n, H * D)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    layer = T.GATLayer(T.DeviceGraph(g), cu(W), cu(a_s), cu(a_d), H, D, slope=0.2, bits=8)
    Hout, _ = layer.forward(cu(X), step=1, layer_id=0)
    dX, dW, das, dad = layer.backward(cu(dY), step=1, layer_id=0)
    torch.cuda.synchronize()
    layer.check_status()
    f = orc.gat_fwd(g, X, W, a_s, a_d, H, D, slope=0.2, bits=8, step=1, layer_id=0, chunk=256)
    eq("H_out", Hout, f["Hout"])
    b = orc.gat_bwd(g, f, X, W, a_s, a_d, dY)
    eq("dH", dX, b["dH"])
    eq("dW", dW, b["dW"])
    bound = 4096 * 2.0 ** -24
    err = np.abs(das.cpu().numpy().astype(np.float64) - b["da_src"])
    assert np.all(err <= bound * b["da_src_abs"] + 1e-7)


@pytest.mark.skipif(not __import__("os").environ.get("TANGO_FULL_REDDIT"),
                    reason="set TANGO_FULL_REDDIT=1 (about 4 min: graph build + oracle on 114 M edges)")
def test_gat_layer_reddit_full_size(T, orc):
    """BASELINE.json configs[3] on one GPU, exactly as bench.py times it (Reddit-shaped: N = 233 K,
    E = 114 M, mean in-degree 489, F = 602, 4 x 128, the v6 dataflow): every output of the layer
    against the full oracle, bit for bit (∂a included: the pinned chunk order of R39)."""
    kw, F, H, D = inputs.WORKLOADS["reddit"]
    g = inputs.workload_graph("reddit")
    W, a_s, a_d = inputs.gat_params(F, H, D)
    X = inputs.features(g.n, F)
    dY = inputs.grad_out(g.n, H * D)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    layer = T.GATLayer(T.DeviceGraph(g), cu(W), cu(a_s), cu(a_d), H, D, slope=0.2, bits=8)
    Hout, amax_out = layer.forward(cu(X), step=0, layer_id=0)
    fv = layer.view()
    dX, dW, das, dad = layer.backward(cu(dY), step=0, layer_id=0)
    bv = layer.view()
    torch.cuda.synchronize()
    layer.check_status()
    assert fv["dataflow"] == 2
    f = orc.gat_fwd(g, X, W, a_s, a_d, H, D, slope=0.2, bits=8, step=0, layer_id=0, chunk=256)
    for name, key in (("qH", "qH"), ("qHp", "qHp"), ("S", "S"), ("qS", "qS"), ("qD", "qD"), ("m", "m"),
                      ("den", "den")):
        eq(name, fv[name], f[key])
    eq("H_out", Hout, f["Hout"])
    eq("amax_out", amax_out, f["amax_out"])
    b = orc.gat_bwd(g, f, X, W, a_s, a_d, dY)
    eq("qG", bv["qG"], b["qG"])
    eq("dalpha_out", bv["dalpha_out"], b["dalpha"][g.out_eid])
    for name in ("P", "dD", "dS", "dHp", "qdHp"):
        eq(name, bv[name], b[name])
    eq("dH", dX, b["dH"])
    eq("dW", dW, b["dW"])
    eq("da_src", das, b["da_src"])
    eq("da_dst", dad, b["da_dst"])
