"""GPU parity of the NEXT-4 sub-byte path (P:1219-1246 INT4 SDDMM): packed 4-bit
SR quantization (tango_quantize_int4) against the oracle's bits = 4 codes, and the warp-per-row
SDDMM-dot / SDDMM-add on int8 and packed int4 codes (tango_sddmm_qn) against the oracle — bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2308_00890_b200 import inputs  # noqa: E402
from test_gpu_layer import cu, eq  # noqa: E402


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2308_00890_b200 import tango
    tango.load()
    return tango


def unpack4(q, cols):
    """packed nibbles (test-side bit unpacking) -> int8 codes [rows][cols]"""
    b = q.cpu().numpy().astype(np.uint8)[:, : cols // 2]
    lo = (b & 0xF).astype(np.int8)
    hi = (b >> 4).astype(np.int8)
    out = np.empty((b.shape[0], cols), np.int8)
    out[:, 0::2], out[:, 1::2] = lo, hi
    return np.where(out >= 8, out - 16, out).astype(np.int8)


@pytest.mark.parametrize("rows,cols,row0", [(1000, 256, 0), (37, 8, 5), (64, 512, 3)])
def test_quantize_int4_parity(T, orc, rows, cols, row0):
    x = inputs.features(rows, cols, seed=51)
    q, s, am = T.quantize_int4(cu(x), seed=9, step=4, tag=0x105, global_row0=row0)
    torch.cuda.synchronize()
    want, ws, wam = orc.quantize(x, 4, seed=9, step=4, tag=0x105, g0=row0 * cols)
    assert np.array_equal(unpack4(q, cols), want)
    assert s.item() == ws and am.item() == wam
    assert np.abs(want).max() <= 7


CASES = [((64, 256, 0), 4, 16, 256), ((2000, 12000, 1), 4, 64, 256), ((500, 2000, 2), 2, 128, 7),
         ((300, 900, 3), 1, 32, 256)]


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("gspec,heads,D,chunk", CASES)
def test_sddmm_dot_qn_parity(T, orc, bits, gspec, heads, D, chunk):
    n, d, s = gspec
    gr = inputs.random_graph(n, d, seed=s)
    dg = T.DeviceGraph(gr, chunk=chunk)
    cols = heads * D
    A = inputs.features(gr.n, cols, seed=s + 10)
    B = inputs.features(gr.n, cols, seed=s + 11)
    qa_w, sa_w, _ = orc.quantize(A, bits, seed=1, tag=6)
    qb_w, sb_w, _ = orc.quantize(B, bits, seed=1, tag=3)
    if bits == 4:
        qa, sa, _ = T.quantize_int4(cu(A), seed=1, tag=6)
        qb, sb, _ = T.quantize_int4(cu(B), seed=1, tag=3)
        assert np.array_equal(unpack4(qa, cols), qa_w) and np.array_equal(unpack4(qb, cols), qb_w)
    else:
        qa, sa, _ = T.quantize(cu(A), bits=8, seed=1, tag=6, ld=cols)
        qb, sb, _ = T.quantize(cu(B), bits=8, seed=1, tag=3, ld=cols)
    out, _ = T.sddmm_qn(dg, T.TANGO_SDDMM_DOT, bits, qb, sb, qa, sa, heads, cols)
    torch.cuda.synchronize()
    want = orc.sddmm_dot(gr, heads, cols, orc.qref(qa_w, s=sa_w), orc.qref(qb_w, s=sb_w), chunk=chunk)
    eq(f"sddmm_dot int{bits}", out, want)


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("gspec,heads", [((64, 256, 0), 4), ((2000, 12000, 1), 4), ((300, 900, 3), 2)])
def test_sddmm_add_qn_parity(T, orc, bits, gspec, heads):
    n, d, s = gspec
    gr = inputs.random_graph(n, d, seed=s)
    if gr.n * heads % 8:
        pytest.skip("flat int4 packing needs n*heads % 8 == 0")
    dg = T.DeviceGraph(gr)
    S = inputs.features(gr.n, heads, seed=s + 20)
    Dm = inputs.features(gr.n, heads, seed=s + 21)
    qs_w, ss_w, _ = orc.quantize(S, bits, seed=2, tag=4)
    qd_w, sd_w, _ = orc.quantize(Dm, bits, seed=2, tag=5)
    if bits == 4:   # [n][heads] packed as one flat run (same element index g, same bytes)
        flat = lambda a: cu(a.reshape(-1, 8))
        qs, ss, _ = T.quantize_int4(flat(S), seed=2, tag=4, ld_bytes=4)
        qd, sd, _ = T.quantize_int4(flat(Dm), seed=2, tag=5, ld_bytes=4)
        qs, qd = qs.reshape(gr.n, heads // 2), qd.reshape(gr.n, heads // 2)
    else:
        qs, ss, _ = T.quantize(cu(S), bits=8, seed=2, tag=4, ld=heads)
        qd, sd, _ = T.quantize(cu(Dm), bits=8, seed=2, tag=5, ld=heads)
    e_pre, el = T.sddmm_qn(dg, T.TANGO_SDDMM_ADD, bits, qs, ss, qd, sd, heads, heads, slope=0.2)
    torch.cuda.synchronize()
    we, wl = orc.sddmm_add(gr, heads, orc.qref(qs_w, s=ss_w), orc.qref(qd_w, s=sd_w), 0.2)
    eq("e_pre", e_pre, we)
    eq("el", el, wl)
