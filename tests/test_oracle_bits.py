"""Oracle pins for the bit-width derivation (NEXT-2): Error_X (§3.2 Eq.4,
reading A24 denominator) and select_bits (threshold 0.3, reading R31 nearest rounding)."""
import numpy as np
import pytest


def test_error_term_closed_forms(orc):
    assert orc.error_term(1.25, 1.25) == 0.0                 # no rounding error -> 0
    assert orc.error_term(0.0, 0.0) == 0.0                   # ε guards X = X̂ = 0
    assert orc.error_term(1.0, 0.0) == np.float32(1.0) / np.float32(1.0005)
    # reading A24: |X| + |X̂| + ε; the printed X + X̂ + ε would give 0.0003/0.0002 = 1.5 here
    assert orc.error_term(-0.0003, 0.0) == np.float32(0.0003) / np.float32(np.float32(0.0003) + np.float32(0.0005))
    assert orc.error_term(-2.0, -1.0) == np.float32(1.0) / np.float32(3.0005)


def test_error_term_range(orc):
    rng = np.random.default_rng(1)
    for x, xh in rng.standard_normal((2000, 2)).astype(np.float32):
        t = orc.error_term(x, xh)
        assert 0.0 <= t <= 1.0                                # P:495 "value range [0, 1]"


def test_error_x_exact_grid_and_zeros(orc):
    e = 3
    k = np.arange(-127, 128, dtype=np.float32)
    x = (k * np.float32(2.0 ** -e)).astype(np.float32)       # amax = 127·2^-e -> r = 2^e exactly
    q, s, _ = orc.quantize(x, 8, step=3, tag=9)
    assert np.array_equal(q, k.astype(np.int8))
    assert orc.error_x(x, q, s) == 0.0
    z = np.zeros(1000, np.float32)
    qz, sz, _ = orc.quantize(z, 8)
    assert orc.error_x(z, qz, sz) == 0.0
    assert orc.error_x(z[:0], qz[:0], sz) == 0.0


def test_select_bits_picks_the_grid(orc):
    # values on the 4-bit grid (amax = 7, codes ±7): B = 4 is exact, B = 2, 3 are not
    rng = np.random.default_rng(2)
    x = rng.integers(-7, 8, 5000).astype(np.float32)
    x[0] = 7.0
    bits, errs, none = orc.select_bits(x, threshold=1e-12)
    assert bits == 4 and not none
    assert errs[4 - 2] == 0.0 and errs[0] > 0.3 and errs[1] > 0.0


def test_select_bits_gaussian_monotone_and_threshold(orc):
    x = np.random.default_rng(3).standard_normal(200_000).astype(np.float32)
    bits, errs, none = orc.select_bits(x, threshold=0.3)
    assert np.all(np.diff(errs) < 0)                          # non-increasing in B (SPEC invariant)
    assert np.all((errs >= 0) & (errs <= 1))
    assert errs[bits - 2] <= 0.3 and (bits == 2 or errs[bits - 3] > 0.3)
    b0, e0, none0 = orc.select_bits(x, threshold=0.0)
    assert none0 and b0 == 8
    b1, e1, _ = orc.select_bits(x, threshold=0.3, bmin=5, bmax=7)
    assert np.array_equal(e1, errs[3:6])


def test_select_bits_errors(orc):
    x = np.ones(10, np.float32)
    with pytest.raises(orc.OracleError):
        orc.select_bits(x, bmin=1)
    with pytest.raises(orc.OracleError):
        orc.select_bits(x, bmin=6, bmax=5)
    x[3] = np.nan
    with pytest.raises(orc.OracleError):
        orc.select_bits(x)
