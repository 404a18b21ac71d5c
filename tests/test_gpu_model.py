"""GPU parity of the NEXT-1 path: tango_sgemm, tango_colsum, tango_bias_act_fwd/bwd,
tango_cross_entropy, tango_sgd_update, the FP32 final GAT layer (tango_gat_out_fwd/bwd) and one full
training step of a multi-layer GAT (paper_2308_00890_b200.model.GATModel) against the CPU oracle.

Bit-exact everywhere except: ∂a_src / ∂a_dst (order-free atomics; DESIGN.md §3 bound) and the loss
scalar (logf + double atomics; 1e-6 relative).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2308_00890_b200 import inputs  # noqa: E402
from test_gpu_layer import cu, eq, da_ok  # noqa: E402


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_00890_b200 import tango
    tango.load()
    return tango


def _rand(shape, seed, scale=1.0):
    return (np.random.Generator(np.random.PCG64(seed)).standard_normal(shape) * scale).astype(np.float32)


@pytest.mark.parametrize("M,N,K", [(100, 70, 2500), (1, 1, 1), (65, 63, 1024), (130, 17, 1025), (64, 64, 0),
                                   (3000, 160, 512), (301, 512, 160), (512, 160, 5000), (257, 161, 13),
                                   (40, 300, 7)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_sgemm_parity(T, orc, M, N, K, ta, tb):
    A = _rand((M, K), 1)
    B = _rand((K, N), 2)
    want = orc.sgemm(A.T.copy() if ta else A, B.T.copy() if tb else B, transA=ta, transB=tb)
    Ad = cu(A.T.copy() if ta else A).reshape((K, M) if ta else (M, K))
    Bd = cu(B.T.copy() if tb else B).reshape((N, K) if tb else (K, N))
    got = T.sgemm(Ad, Bd, a_layout=T.TANGO_MN_MAJOR if ta else T.TANGO_K_MAJOR,
                  b_layout=T.TANGO_K_MAJOR if tb else T.TANGO_MN_MAJOR)
    torch.cuda.synchronize()
    eq("sgemm", got, want)


@pytest.mark.parametrize("rows,cols", [(3000, 37), (1, 5), (1024, 300), (2049, 1)])
def test_colsum_and_bias_act_parity(T, orc, rows, cols):
    x = _rand((rows, cols), 3)
    b = _rand(cols, 4)
    a_want, am_want = orc.bias_relu_fwd(x, b)
    a, am = T.bias_act_fwd(cu(x), cu(b))
    eq("act", a, a_want)
    eq("amax act", am[0:1], np.array([am_want]))
    da = _rand((rows, cols), 5)
    dx_want, db_want, amd_want = orc.bias_relu_bwd(a_want, da)
    dx, db, amd = T.bias_act_bwd(a, cu(da))
    eq("dx", dx, dx_want)
    eq("db", db, db_want)
    eq("amax dx", amd[0:1], np.array([amd_want]))
    eq("colsum", T.colsum(cu(x)), orc.colsum(x))
    torch.cuda.synchronize()


@pytest.mark.parametrize("rows,C,frac", [(1000, 40, 0.537), (7, 3, 1.0), (300, 1000, 0.5)])
def test_cross_entropy_parity(T, orc, rows, C, frac):
    z = _rand((rows, C), 6, 3.0)
    lab = inputs.labels(rows, C, train_frac=frac, seed=7)
    n_lab = int((lab >= 0).sum())
    loss_w, dz_w, _ = orc.cross_entropy(z, lab)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    loss, dz = T.cross_entropy(cu(z), cu(lab), n_lab, status=st)
    torch.cuda.synchronize()
    eq("dlogits", dz, dz_w)
    assert abs(loss.item() - loss_w) <= 1e-6 * abs(loss_w)
    assert st.item() == 0
    bad = lab.copy()
    bad[0] = C
    T.cross_entropy(cu(z), cu(bad), n_lab, status=st)
    torch.cuda.synchronize()
    assert st.item() == 1   # TANGO_ERR_INVALID_ARG on the device status word


def test_sgd_parity(T, orc):
    ws = [_rand(s, 10 + i) for i, s in enumerate([(33, 7), (5,), (1000,), (1,)])]
    gs = [_rand(w.shape, 20 + i) for i, w in enumerate(ws)]
    wd = [cu(w) for w in ws]
    T.sgd_update(list(zip(wd, [cu(g) for g in gs])), 0.05)
    torch.cuda.synchronize()
    for w, g, d in zip(ws, gs, wd):
        eq("sgd", d, orc.sgd(w, g, 0.05))


OUT_CASES = [
    # graph (n, draws, seed, self_loops), F, heads, classes, chunk
    ((64, 256, 0, True), 16, 2, 5, 256),
    ((1000, 4000, 2, True), 100, 4, 40, 7),
    ((500, 900, 5, False), 48, 1, 7, 256),
    ((2000, 20000, 6, True), 512, 4, 40, 64),
    ((3000, 30000, 9, True), 64, 8, 100, 5),   # HC = 800 (> 8 columns per lane), chunk 5: most rows heavy
]


@pytest.mark.parametrize("gspec,F,heads,C,chunk", OUT_CASES)
def test_gat_out_layer_parity(T, orc, gspec, F, heads, C, chunk):
    n, d, s, loops = gspec
    gr = inputs.random_graph(n, d, seed=s, self_loops=loops)
    H = _rand((gr.n, F), 31)
    W, a_s, a_d = inputs.gat_params(F, heads, C, seed=32)
    b = _rand(C, 33)
    dz = _rand((gr.n, C), 34, 0.01)
    f = orc.gat_out_fwd(gr, H, W, a_s, a_d, b, heads, C, slope=0.2, chunk=chunk)
    bo = orc.gat_out_bwd(gr, f, H, W, a_s, a_d, dz)
    dg = T.DeviceGraph(gr, chunk=chunk)
    layer = T.GATOutLayer(dg, cu(W), cu(a_s), cu(a_d), cu(b), heads, C, slope=0.2)
    Hd = cu(H)
    logits = layer.forward(Hd)
    dH, dW, das, dad, db = layer.backward(Hd, cu(dz))
    torch.cuda.synchronize()
    v = layer.view()
    eq("Hp", v["Hp"], f["Hp"])
    eq("S", v["S"], f["S"])
    eq("D", v["D"], f["Dd"])
    eq("e_pre", v["e_pre"], f["e_pre"])
    eq("alpha", v["alpha"], f["alpha"])
    eq("m", v["m"], f["m"])
    eq("den", v["den"], f["den"])
    eq("agg", v["agg"], f["agg"])
    eq("logits", logits, f["logits"])
    eq("G", v["G"], bo["G"])
    eq("dalpha", v["dalpha"], bo["dalpha"])
    eq("dE_pre", v["dE_pre"], bo["dE_pre"])
    eq("dD", v["dD"], bo["dD"])
    eq("dS", v["dS"], bo["dS"])
    eq("dHp", v["dHp"], bo["dHp"])
    eq("db", db, bo["db"])
    eq("dH", dH, bo["dH"])
    eq("dW", dW, bo["dW"])
    da_ok(das, bo["da_src"], bo["da_src_abs"])
    da_ok(dad, bo["da_dst"], bo["da_dst_abs"])


MODEL_CASES = [
    # graph, F, heads, head_dim, layers, classes, chunk
    ((300, 1200, 11), 48, 2, 32, 3, 7, 16),
    ((2000, 12000, 12), 128, 4, 128, 3, 40, 256),
    ((500, 2000, 13), 64, 4, 32, 2, 10, 256),
]


@pytest.mark.parametrize("gspec,F,heads,hd,layers,C,chunk", MODEL_CASES)
def test_model_step_parity(T, orc, gspec, F, heads, hd, layers, C, chunk):
    from paper_2308_00890_b200.model import GATModel
    n, d, s = gspec
    gr = inputs.random_graph(n, d, seed=s)
    X = inputs.features(gr.n, F, seed=s + 1)
    hidden, out = inputs.gat_model_params(F, heads, hd, layers, C, bias_scale=0.1, seed=s + 2)
    lab = inputs.labels(gr.n, C, train_frac=0.6, seed=s + 3)
    n_lab = int((lab >= 0).sum())
    lr, step = 0.1, 4
    r = orc.gat_model_step(gr, X, hidden, out, lab, lr=lr, bits=8, step=step, chunk=chunk)
    dg = T.DeviceGraph(gr, chunk=chunk)
    dev = lambda p: {k: (cu(v) if isinstance(v, np.ndarray) else v) for k, v in p.items()}
    hid_d, out_d = [dev(p) for p in hidden], dev(out)
    model = GATModel(dg, hid_d, out_d, slope=0.2, bits=8)
    loss = model.step(cu(X), cu(lab), n_lab, lr, step=step)
    torch.cuda.synchronize()
    model.check_status()
    assert abs(loss.item() - r["loss"]) <= 1e-6 * abs(r["loss"])
    eq("logits", model.logits, r["logits"])
    for l in range(layers - 1):
        eq(f"act{l}", model.act[l], r["hs"][l + 1])
        eq(f"dW{l}", model.grads[l]["W"], r["grads"][l]["W"])
        eq(f"db{l}", model.grads[l]["b"], r["grads"][l]["b"])
        da_ok(model.grads[l]["a_src"], r["grads"][l]["a_src"], r["grads"][l]["da_src_abs"])
        da_ok(model.grads[l]["a_dst"], r["grads"][l]["a_dst"], r["grads"][l]["da_dst_abs"])
        eq(f"W{l} updated", hid_d[l]["W"], r["hidden"][l]["W"])
        eq(f"b{l} updated", hid_d[l]["b"], r["hidden"][l]["b"])
    og = r["out_grads"]
    eq("out dW", model.out_grads["W"], og["W"])
    eq("out db", model.out_grads["b"], og["b"])
    da_ok(model.out_grads["a_src"], og["a_src"], og["da_src_abs"])
    eq("out W updated", out_d["W"], r["out"]["W"])
    eq("out b updated", out_d["b"], r["out"]["b"])


@pytest.mark.parametrize("gspec,F,C,chunk", [((64, 256, 0, True), 16, 5, 256), ((1000, 4000, 2, True), 100, 7, 7),
                                             ((2708, 5278, 3, True), 1433, 7, 256), ((500, 900, 5, False), 48, 40, 3)])
def test_gcn_out_layer_parity(T, orc, gspec, F, C, chunk):
    n, d, s, loops = gspec
    gr = inputs.random_graph(n, d, seed=s, self_loops=loops)
    X = _rand((gr.n, F), 41)
    W = inputs.gcn_params(F, C, seed=42)
    b = _rand(C, 43)
    dz = _rand((gr.n, C), 44, 0.01)
    f = orc.gcn_out_fwd(gr, X, W, b, chunk=chunk)
    bo = orc.gcn_out_bwd(gr, f, X, W, dz)
    layer = T.GCNOutLayer(T.DeviceGraph(gr, chunk=chunk), cu(W), cu(b))
    Xd = cu(X)
    logits = layer.forward(Xd)
    dX, dW, db = layer.backward(Xd, cu(dz))
    torch.cuda.synchronize()
    v = layer.view()
    for k in ("Y", "Ys", "agg"):
        eq(k, v[k], f[k])
    eq("logits", logits, f["logits"])
    for k in ("Gs", "aggb", "dY"):
        eq(k, v[k], bo[k])
    eq("db", db, bo["db"])
    eq("dX", dX, bo["dX"])
    eq("dW", dW, bo["dW"])


@pytest.mark.parametrize("gspec,F,hid,layers,C,chunk", [((2708, 5278, 3), 1433, 128, 2, 7, 256),
                                                       ((400, 1500, 4), 64, 32, 3, 5, 5)])
def test_gcn_model_step_parity(T, orc, gspec, F, hid, layers, C, chunk):
    from paper_2308_00890_b200.model import GCNModel
    n, d, s = gspec
    gr = inputs.random_graph(n, d, seed=s)
    X = inputs.features(gr.n, F, seed=s + 1)
    hidden, out = inputs.gcn_model_params(F, hid, layers, C, bias_scale=0.1, seed=s + 2)
    lab = inputs.labels(gr.n, C, train_frac=0.5, seed=s + 3)
    n_lab = int((lab >= 0).sum())
    r = orc.gcn_model_step(gr, X, hidden, out, lab, lr=0.2, bits=8, step=3, chunk=chunk)
    dev = lambda p: {k: cu(v) for k, v in p.items()}
    hid_d, out_d = [dev(p) for p in hidden], dev(out)
    model = GCNModel(T.DeviceGraph(gr, chunk=chunk), hid_d, out_d, bits=8)
    loss = model.step(cu(X), cu(lab), n_lab, 0.2, step=3)
    torch.cuda.synchronize()
    model.check_status()
    assert abs(loss.item() - r["loss"]) <= 1e-6 * abs(r["loss"])
    eq("logits", model.logits, r["logits"])
    for l in range(layers - 1):
        eq(f"act{l}", model.act[l], r["hs"][l + 1])
        eq(f"dW{l}", model.grads[l]["W"], r["grads"][l]["W"])
        eq(f"db{l}", model.grads[l]["b"], r["grads"][l]["b"])
        eq(f"W{l} updated", hid_d[l]["W"], r["hidden"][l]["W"])
    eq("out dW", model.out_grads["W"], r["out_grads"]["W"])
    eq("out W updated", out_d["W"], r["out"]["W"])
    eq("out b updated", out_d["b"], r["out"]["b"])


def test_cross_entropy_no_labels_and_empty(T, orc):
    # no labelled row: zero loss and zero gradient on both sides
    z = _rand((50, 7), 71)
    lab = np.full(50, -1, np.int32)
    loss_w, dz_w, _ = orc.cross_entropy(z, lab, n_lab=0)
    loss, dz = T.cross_entropy(cu(z), cu(lab), 0)
    torch.cuda.synchronize()
    eq("dlogits", dz, dz_w)
    assert loss.item() == 0.0 and loss_w == 0.0


def test_bias_act_and_sgd_zero_sizes(T):
    x = torch.empty((0, 16), device="cuda")
    y, am = T.bias_act_fwd(x, torch.zeros(16, device="cuda"))
    dx, db, amd = T.bias_act_bwd(y, x)
    torch.cuda.synchronize()
    assert am.item() == 0.0 and amd.item() == 0.0 and torch.all(db == 0)
    T.sgd_update([], 0.1)
