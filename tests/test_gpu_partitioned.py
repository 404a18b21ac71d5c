"""The partitioned (multi-GPU) path on ONE GPU: P ranks as host threads with an in-process loopback
communicator (tango_comm_init_local; same collective semantics as the NCCL communicator), each
rank owning a destination-row block.  This runs every kernel with row_begin > 0,
the source pass's recompute path (no out_eid on a partitioned graph) and every collective of
the layer; the concatenated per-rank outputs must equal the single-process oracle bit for bit
(∂a within the derived bound).
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2308_00890_b200 import inputs  # noqa: E402
from paper_2308_00890_b200.partition import partition_rows  # noqa: E402


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_00890_b200 import tango
    tango.load()
    return tango


CASES = [  # P, graph (n, draws, seed), F, heads, head_dim, chunk
    (2, (1500, 12000, 3), 64, 4, 32, 16),
    (3, (2000, 20000, 4), 128, 4, 128, 256),
    (4, (900, 6000, 5), 40, 2, 32, 7),
]


@pytest.mark.parametrize("case", CASES, ids=[f"P{c[0]}" for c in CASES])
def test_gat_partitioned_local_comm(T, orc, case):
    P, (n, draws, seed), F, heads, hd, chunk = case
    gr = inputs.chung_lu_graph(n, draws, 2.1, dmax=n // 3, seed=seed)
    HD = heads * hd
    X = inputs.features(gr.n, F, seed=21)
    W, a_s, a_d = inputs.gat_params(F, heads, hd, seed=22)
    dY = inputs.grad_out(gr.n, HD, seed=23)
    step, layer_id = 5, 2
    starts = partition_rows(gr, P)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    Wd, asd, add = cu(W), cu(a_s), cu(a_d)
    group = T.LocalGroup(P)
    res, err = [None] * P, [None] * P

    def rank(r):
        try:
            rb, re = starts[r], starts[r + 1]
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                dg = T.DeviceGraph(gr, chunk=chunk, row_begin=rb, row_end=re)
                comm = T.Comm.local(group, r, starts)
                layer = T.GATLayer(dg, Wd, asd, add, heads, hd, slope=0.2, bits=8, comm=comm)
                Hout, amax = layer.forward(cu(X[rb:re]), step=step, layer_id=layer_id)
                dX, dW, das, dad = layer.backward(cu(dY[rb:re]), step=step, layer_id=layer_id)
                s.synchronize()
                layer.check_status()
                res[r] = [t.cpu().numpy() for t in (Hout, amax, dX, dW, das, dad)]
                comm.close()
        except Exception as e:   # surfaced below
            err[r] = e

    ths = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(P)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    group.close()
    for e in err:
        if e is not None:
            raise e

    f = orc.gat_fwd(gr, X, W, a_s, a_d, heads, hd, slope=0.2, bits=8, step=step, layer_id=layer_id, chunk=chunk)
    b = orc.gat_bwd(gr, f, X, W, a_s, a_d, dY)
    Hout = np.concatenate([r[0] for r in res])
    dX = np.concatenate([r[2] for r in res])
    assert np.array_equal(Hout, f["Hout"]), np.argwhere(Hout != f["Hout"])[:3]
    assert np.array_equal(dX, b["dH"]), np.argwhere(dX != b["dH"])[:3]
    for r in range(P):
        assert np.array_equal(res[r][1], np.asarray(f["amax_out"]).reshape(1)), r   # AllReduce-MAX
        assert np.array_equal(res[r][3], b["dW"]), r                               # int64 AllReduce-SUM
        bound = 4096 * 2.0 ** -24
        for got, want, absum in ((res[r][4], b["da_src"], b["da_src_abs"]), (res[r][5], b["da_dst"], b["da_dst_abs"])):
            assert np.all(np.abs(got.astype(np.float64) - want) <= bound * absum + 1e-7), r


@pytest.mark.parametrize("P", [2, 3])
def test_gcn_partitioned_local_comm(T, orc, P):
    gr = inputs.chung_lu_graph(1200, 9000, 2.3, dmax=400, seed=8)
    F, O = 96, 40
    X = inputs.features(gr.n, F, seed=31)
    W = inputs.gcn_params(F, O, seed=32)
    dY = inputs.grad_out(gr.n, O, seed=33)
    starts = partition_rows(gr, P)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    Wd = cu(W)
    group = T.LocalGroup(P)
    res, err = [None] * P, [None] * P

    def rank(r):
        try:
            rb, re = starts[r], starts[r + 1]
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                dg = T.DeviceGraph(gr, row_begin=rb, row_end=re)
                comm = T.Comm.local(group, r, starts)
                layer = T.GCNLayer(dg, Wd, bits=8, comm=comm)
                out, _ = layer.forward(cu(X[rb:re]), step=1, layer_id=0)
                dX, dW = layer.backward(cu(dY[rb:re]), step=1, layer_id=0)
                s.synchronize()
                layer.check_status()
                res[r] = [t.cpu().numpy() for t in (out, dX, dW)]
                comm.close()
        except Exception as e:
            err[r] = e

    ths = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(P)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    group.close()
    for e in err:
        if e is not None:
            raise e
    f = orc.gcn_fwd(gr, X, W, bits=8, step=1, layer_id=0)
    b = orc.gcn_bwd(gr, f, X, W, dY)
    assert np.array_equal(np.concatenate([r[0] for r in res]), f["out"])
    assert np.array_equal(np.concatenate([r[1] for r in res]), b["dX"])
    for r in range(P):
        assert np.array_equal(res[r][2], b["dW"]), r


@pytest.mark.parametrize("staged", [True, False], ids=["padded_allgather", "grouped_broadcast"])
def test_nccl_single_rank_comm(T, orc, staged):
    """The NCCL transport itself (tango_comm_init over a real ncclComm, nranks = 1, set to always run its
    collectives): every collective of the GAT and GCN layers is enqueued through NCCL on the caller's
    stream (counted by tango_comm_nccl_calls), node-row all-gathers as one padded ncclAllGather through
    the reserved staging buffer or as grouped broadcasts; the results must equal the oracle bit for bit
    (∂a within the bound).  gpurun provides one GPU, so this is the NCCL path's only on-device check; the
    multi-rank dataflow is covered by the loopback and gloo tests."""
    from test_gpu_layer import da_ok, eq
    gr = inputs.random_graph(1200, 6000, seed=31)
    F, heads, hd = 64, 4, 32
    X = inputs.features(gr.n, F, seed=32)
    W, a_s, a_d = inputs.gat_params(F, heads, hd, seed=33)
    dY = inputs.grad_out(gr.n, heads * hd, seed=34)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    comm = T.Comm(1, 0, T.Comm.unique_id(), [0, gr.n], always=True, reserve_row_bytes=512 if staged else 0)
    try:
        dg = T.DeviceGraph(gr, chunk=16, row_begin=0, row_end=gr.n)
        layer = T.GATLayer(dg, cu(W), cu(a_s), cu(a_d), heads, hd, slope=0.2, bits=8, comm=comm)
        Hout, _ = layer.forward(cu(X), step=3, layer_id=1)
        dX, dW, das, dad = layer.backward(cu(dY), step=3, layer_id=1)
        Wg = inputs.gcn_params(F, 48, seed=35)
        gl = T.GCNLayer(dg, cu(Wg), bits=8, comm=comm)
        gout, _ = gl.forward(cu(X), step=3, layer_id=2)
        gdX, gdW = gl.backward(cu(dY[:, :48]), step=3, layer_id=2)
        torch.cuda.synchronize()
        layer.check_status()
        calls = comm.nccl_calls()
    finally:
        comm.close()
    # GAT fwd: amax(H), {amax H', S, D}, q_H', q_S, q_D, amax(out), m, den; bwd: amax(dH_out), q_G, P,
    # amax(dH'), dW, da_src, da_dst (+ amax(dH)); GCN adds its own: all of them must have executed
    assert calls >= 20, calls
    f = orc.gat_fwd(gr, X, W, a_s, a_d, heads, hd, slope=0.2, bits=8, step=3, layer_id=1, chunk=16)
    b = orc.gat_bwd(gr, f, X, W, a_s, a_d, dY)
    eq("H_out", Hout, f["Hout"])
    eq("dH", dX, b["dH"])
    eq("dW", dW, b["dW"])
    da_ok(das, b["da_src"], b["da_src_abs"])
    gf = orc.gcn_fwd(gr, X, Wg, bits=8, step=3, layer_id=2, chunk=16)
    gb = orc.gcn_bwd(gr, gf, X, Wg, dY[:, :48])
    eq("gcn out", gout, gf["out"])
    eq("gcn dX", gdX, gb["dX"])
    eq("gcn dW", gdW, gb["dW"])
