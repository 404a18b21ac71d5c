"""Pins for the oracle's Philox stream, quantizer, pinned exp and integer GEMM.

Everything here checks the oracle against something other than itself:
published known-answer vectors, closed forms, statistics, the paper's Fig.4
integer fragment, and numpy's integer matmul (a library routine).
"""
import math

import numpy as np
import pytest


# Random123 known-answer vectors for philox4x32_10 (kat_vectors in the Random123 distribution).
KAT = [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_kat(orc, ctr, key, want):
    assert [int(x) for x in orc.philox(ctr, key)] == want


def test_sr_uniform_halfword_layout(orc):
    # element g uses half-word (g & 7) of Philox(ctr={g>>3, 0, tag, step}, key=seed) (reading R4)
    seed, step, tag = 0x1234_5678_9ABC, 7, 0x305
    for g in [0, 1, 2, 7, 8, 15, 1_000_003, (1 << 35) + 5]:
        blk = g >> 3
        w = orc.philox([blk & 0xFFFFFFFF, blk >> 32, tag, step], [seed & 0xFFFFFFFF, seed >> 32])
        j = g & 7
        word = int(w[j >> 1])
        hw = (word >> 16) if (j & 1) else (word & 0xFFFF)
        assert orc.sr_uniform(seed, step, tag, g) == hw / 65536.0


def test_sr_uniform_statistics(orc):
    u = np.array([orc.sr_uniform(99, 0, 1, g) for g in range(20000)])
    assert u.min() >= 0.0 and u.max() < 1.0
    assert np.all(u * 65536 == np.floor(u * 65536))           # 16-bit grid
    assert abs(u.mean() - 0.5) < 3 * math.sqrt(1 / 12 / u.size)


def test_quantize_exact_grid(orc):
    # X = k * 2^-e with amax = 127 * 2^-e  =>  r = 2^e exactly, x = k exactly, q = k for any u.
    rng = np.random.default_rng(0)
    k = rng.integers(-127, 128, size=4096).astype(np.float32)
    k[0] = 127.0
    for e in (0, 3, 10):
        x = (k * np.float32(2.0 ** -e)).astype(np.float32)
        for seed in (0, 1, 12345):
            q, s, amax = orc.quantize(x, 8, seed=seed, tag=3)
            assert np.array_equal(q.astype(np.float32), k)
            assert s == np.float32(127 * 2.0 ** -e) / np.float32(127)


def test_quantize_endpoints_and_zero(orc):
    x = np.array([-2.5, 2.5, 0.0, 1.0], np.float32)
    q, s, amax = orc.quantize(x, 8)
    assert q[0] == -127 and q[1] == 127 and q[2] == 0
    assert amax == np.float32(2.5) and s == np.float32(2.5) / np.float32(127)
    q, s, amax = orc.quantize(np.zeros(100, np.float32), 8)
    assert np.all(q == 0) and s == 1.0 and amax == 0.0


@pytest.mark.parametrize("bits", [2, 3, 4, 6, 8])
def test_quantize_range_and_error_bound(orc, bits):
    rng = np.random.default_rng(bits)
    x = rng.standard_normal(50_000).astype(np.float32) * 3
    q, s, amax = orc.quantize(x, bits, seed=5, tag=1)
    qmax = 2 ** (bits - 1) - 1
    assert q.min() >= -qmax and q.max() <= qmax
    assert np.all(np.abs(q.astype(np.float64) * s - x) < s * (1 + 1e-6))   # SR moves at most one step
    # floor/ceil only: q in {floor(x r), floor(x r)+1}
    xr = x.astype(np.float64) * (qmax / amax)
    assert np.all((q >= np.floor(xr) - 1e-3) & (q <= np.floor(xr) + 1 + 1e-3))


def test_quantize_unbiased(orc):
    # Eq.3: E[q] = x.  All elements equal -> independent draws; amax fixed by override.
    n = 100_000
    x = np.full(n, 0.3, np.float32)
    q, s, _ = orc.quantize(x, 8, seed=77, tag=2, amax=np.float32(1.0))
    target = float(np.float32(0.3) * (np.float32(127.0) / np.float32(1.0)))
    fr = target - math.floor(target)
    assert abs(q.mean() - target) < 3 * math.sqrt(fr * (1 - fr) / n) + 2 ** -16
    # P(round up) = fr (u has 16-bit resolution: bias <= 2^-16)
    assert set(np.unique(q)) <= {math.floor(target), math.floor(target) + 1}


def test_quantize_errors(orc):
    x = np.array([1.0, np.nan], np.float32)
    with pytest.raises(orc.OracleError):
        orc.quantize(x, 8)
    with pytest.raises(orc.OracleError):
        orc.quantize(np.array([np.inf], np.float32), 8)
    with pytest.raises(orc.OracleError):
        orc.quantize(np.ones(3, np.float32), 9)


def test_quantize_global_index_offset(orc):
    # counter = global element index: quantizing a slice with g0 equals the slice of the whole (partition invariance)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((50, 7)).astype(np.float32)
    q, s, amax = orc.quantize(x, 8, seed=9, tag=4)
    q2, s2, _ = orc.quantize(x[20:35], 8, seed=9, tag=4, g0=20 * 7, amax=amax)
    assert s2 == s and np.array_equal(q2, q[20:35])


def test_exp_p(orc):
    assert orc.exp_p(0.0) == 1.0
    xs = np.linspace(-86.0, 0.0, 20001).astype(np.float32)
    got = np.array([orc.exp_p(x) for x in xs], np.float64)
    ref = np.exp(xs.astype(np.float64))
    assert np.max(np.abs(got - ref) / ref) < 4e-6
    assert np.all(np.diff(got) >= 0)                    # monotone on the grid
    assert orc.exp_p(-200.0) == 0.0


def test_gemm_fig4_fragment(orc):
    import json, os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "toy_gat.json")))
    a = np.array([gold["fig4_qH_row0"]["value"]], np.int8)             # 1 x 4
    b = np.array(gold["fig4_qW_col0"]["value"], np.int8).reshape(4, 1)  # 4 x 1
    acc, accf = orc.gemm(orc.qref(q=a), orc.qref(q=b), 1, 1, 4, 4, 1)
    assert acc[0, 0] == gold["fig4_dot"]["value"] == 11781
    assert acc[0, 0] > 127                                              # "exceed the 8-bit range"


@pytest.mark.parametrize("transA,transB", [(False, False), (True, False), (False, True)])
def test_gemm_bruteforce(orc, transA, transB):
    rng = np.random.default_rng(11)
    M, N, K = 37, 29, 301
    A = rng.integers(-127, 128, size=(M, K)).astype(np.int8)
    B = rng.integers(-127, 128, size=(K, N)).astype(np.int8)
    As = A.T.copy() if transA else A
    Bs = B.T.copy() if transB else B
    acc, accf = orc.gemm(orc.qref(q=As), orc.qref(q=Bs), M, N, K, As.shape[1], Bs.shape[1], transA, transB)
    ref = A.astype(np.int64) @ B.astype(np.int64)
    assert np.array_equal(acc, ref)
    assert np.array_equal(accf, ref.astype(np.float32))


def test_int32_bound():
    # reading R27: 127^2 * K < 2^31 holds up to K = 133,144 (forward and dH GEMMs), not for dW (K = N).
    assert 127 * 127 * 133_144 < 2 ** 31 <= 127 * 127 * 133_145
