"""GPU parity of the bit-width derivation (NEXT-2): tango_quant_error and tango_select_bits vs the
oracle.  Terms are fp32 and bit-identical; the fp64 sums differ only in order (relative 1e-12)."""
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


@pytest.mark.parametrize("shape", [(1, 1), (37, 53), (1000, 128), (20000, 512)])
def test_quant_error_parity(T, orc, shape):
    x = inputs.features(shape[0], shape[1], seed=shape[0])
    xd = torch.from_numpy(x).cuda()
    q, s, _ = T.quantize(xd, bits=8, seed=5, step=2, tag=7)
    got = float(T.quant_error(xd, q, s).item())
    qo, so, _ = orc.quantize(x, 8, seed=5, step=2, tag=7)
    want = orc.error_x(x, qo, so)
    assert np.array_equal(q[:, :shape[1]].cpu().numpy(), qo)
    assert abs(got - want) <= 1e-12 * max(1.0, abs(want)), (got, want)


@pytest.mark.parametrize("case", ["gauss", "grid4", "hout"])
def test_select_bits_parity(T, orc, case):
    rng = np.random.default_rng(11)
    if case == "gauss":
        x = rng.standard_normal(300_000).astype(np.float32)
    elif case == "grid4":
        x = rng.integers(-7, 8, 100_000).astype(np.float32)
    else:   # a first-layer GAT output (the tensor P:513 applies the rule to)
        g = inputs.random_graph(3000, 30000, seed=12)
        W, a_s, a_d = inputs.gat_params(64, 4, 32, seed=13)
        layer = T.GATLayer(T.DeviceGraph(g), torch.from_numpy(W).cuda(), torch.from_numpy(a_s).cuda(),
                           torch.from_numpy(a_d).cuda(), 4, 32)
        hout, _ = layer.forward(torch.from_numpy(inputs.features(g.n, 64, seed=14)).cuda())
        x = hout.cpu().numpy().ravel()
    for thr in (0.3, 1e-12, 0.05):
        bits, errs = T.select_bits(torch.from_numpy(x).cuda(), threshold=thr)
        b_o, e_o, none = orc.select_bits(x, threshold=thr)
        e = errs.cpu().numpy()
        assert np.all(np.abs(e - e_o) <= 1e-12 * np.maximum(1.0, np.abs(e_o))), (e, e_o)
        assert int(bits.item()) == (-b_o if none else b_o)
