"""Oracle pins: fixed-point multiplier, requantize (Eq. 5).

Each test pins the oracle to something other than itself: SPEC worked
examples (tests/golden/spec_examples.json), closed forms (exact power-of-two
scales), invariants of the rounding definitions, and an error bound against
the real-valued ratio.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ----------------------------------------------------------------------------- multiplier
@pytest.mark.parametrize("ex", GOLD["derive_multiplier"], ids=lambda e: str(e["m"]))
def test_multiplier_spec_examples(orc, ex):
    M, shift = orc.derive_multiplier(ex["m"])
    assert M == ex["M"] and shift == -ex["spec_s"]


@pytest.mark.parametrize("m,M,shift", [
    (0.5, 1073741824, 0), (1.0, 1073741824, 1), (0.25, 1073741824, -1),
    # 0.1 = 0.8 * 2^-3; 0.8 * 2^31 = 1717986918.4 -> 1717986918
    (0.1, 1717986918, -3),
    # 1/3 = (2/3) * 2^-1; (2/3) * 2^31 = 1431655765.33 -> 1431655765
    (1.0 / 3.0, 1431655765, -1),
    # fl32(0.1) = 13421773 * 2^-27; sig*2^31 = 13421773 * 2^7 = 1717986944 exactly
    (float(np.float32(0.1)), 1717986944, -3),
])
def test_multiplier_closed_forms(orc, m, M, shift):
    assert orc.derive_multiplier(m) == (M, shift)


def test_multiplier_tie_rounds_half_away(orc):
    # m = 0.5 + 2^-32: sig * 2^31 = 2^30 + 0.5 exactly; half-away -> 2^30 + 1
    # (Python's round() would give 2^30 -- the oracle must not use it; reading R2)
    assert orc.derive_multiplier(0.5 + 2.0 ** -32) == (2 ** 30 + 1, 0)


def test_multiplier_carry_renormalises(orc):
    # sig just below 1 rounds up to 2^31 -> renormalised to (2^30, e+1)
    m = 1.0 - 2.0 ** -40
    assert orc.derive_multiplier(m) == (2 ** 30, 1)


def test_multiplier_relative_error_bound(orc):
    g = np.random.default_rng(7)
    for m in np.exp(g.uniform(-30, 10, size=2000)):
        M, s = orc.derive_multiplier(float(m))
        assert 2 ** 30 <= M < 2 ** 31
        approx = Fraction(M) * Fraction(2) ** (s - 31)
        # |m - M*2^(s-31)| <= 1/2 ulp of the 31-bit significand
        assert abs(Fraction(float(m)) - approx) <= Fraction(2) ** (s - 32)


@pytest.mark.parametrize("bad", [0.0, -1.0, float("nan"), float("inf")])
def test_multiplier_rejects(orc, bad):
    with pytest.raises(ValueError):
        orc.derive_multiplier(bad)


# ----------------------------------------------------------------------------- rounding
@pytest.mark.parametrize("ex", GOLD["apply_fixed_point"], ids=lambda e: f'{e["x"]}')
def test_round_spec_examples(orc, ex):
    M, s = orc.derive_multiplier(ex["m"])
    assert orc.round_fixed(ex["x"], M, s, ex["mode"]) == ex["y"]


@pytest.mark.parametrize("x,up,near", [(5, 3, 3), (-5, -2, -3), (3, 2, 2), (-3, -1, -2), (4, 2, 2), (-4, -2, -2),
                                       (1, 1, 1), (-1, 0, -1), (0, 0, 0)])
def test_round_ties_at_half(orc, x, up, near):
    # m = 0.5 exactly: x/2 has ties at odd x; UPWARD -> toward +inf, TONEAREST -> away from 0 (reading R1)
    M, s = orc.derive_multiplier(0.5)
    assert orc.round_fixed(x, M, s, "upward") == up
    assert orc.round_fixed(x, M, s, "tonearest") == near


def test_round_power_of_two_is_exact(orc):
    # m = 2^j: x*m is exact when j >= 0, and for j < 0 the result is the nearest integer of x/2^-j
    g = np.random.default_rng(1)
    for j in range(-20, 8):
        M, s = orc.derive_multiplier(2.0 ** j)
        for x in g.integers(-2 ** 31, 2 ** 31, size=50):
            x = int(x)
            q = Fraction(x) * Fraction(2) ** j
            up = orc.round_fixed(x, M, s, "upward")
            if q.denominator == 1:
                assert up == q
            else:
                assert abs(up - q) <= Fraction(1, 2)


def test_round_invariants(orc):
    """Invariants of the two rounding definitions (no formula retyped):
    |R(q) - q| <= 1/2; TONEAREST is odd-symmetric; UPWARD commutes with integer
    translation by whole multiples of the denominator; both are monotone."""
    g = np.random.default_rng(2)
    for _ in range(300):
        m = float(np.exp(g.uniform(-20, 2)))
        M, s = orc.derive_multiplier(m)
        xs = np.sort(g.integers(-2 ** 31, 2 ** 31, size=40))
        prev_u = prev_n = None
        for x in xs:
            x = int(x)
            q = Fraction(x * M) / Fraction(2) ** (31 - s)
            u = orc.round_fixed(x, M, s, "upward")
            n = orc.round_fixed(x, M, s, "tonearest")
            assert abs(u - q) <= Fraction(1, 2) and abs(n - q) <= Fraction(1, 2)
            assert orc.round_fixed(-x, M, s, "tonearest") == -n
            if (q - math.floor(q)) != Fraction(1, 2):
                assert u == n          # the modes differ only on exact ties
            if prev_u is not None:
                assert u >= prev_u and n >= prev_n
            prev_u, prev_n = u, n
        k = 31 - s
        if 0 < k < 62:
            x = int(xs[0])
            assert orc.round_fixed(x + 2 ** k, M, s, "upward") == orc.round_fixed(x, M, s, "upward") + M


# ----------------------------------------------------------------------------- requantize
@pytest.mark.parametrize("ex", GOLD["requantize"], ids=lambda e: f'{e["q"]}')
def test_requantize_spec_examples(orc, ex):
    y = orc.requantize(np.array([ex["q"]], np.int32), [ex["s_in"]], ex["zp_in"], ex["s_out"], ex["zp_out"], "s32")
    assert int(y[0]) == ex["y"]


def test_requantize_identity_when_scales_equal(orc):
    # scale_A = scale_B, zp_A = zp_B -> Q_B = clamp(Q_A)
    x = np.arange(-128, 128, dtype=np.int32)
    y = orc.requantize(x, [0.37], 5, 0.37, 5, "s8")
    assert np.array_equal(y.astype(np.int64), np.clip(x, -128, 127))


def test_requantize_fixed_vs_real_ratio(orc):
    """|fixed-point result - exactly rounded real-ratio result| <= 1, and == 0
    for power-of-two ratios (256 codes x 50 scale triples + 10k int32)."""
    g = np.random.default_rng(3)
    for t in range(50):
        s_in = np.float32(g.uniform(1e-3, 1.0))
        s_out = np.float32(g.uniform(1e-3, 1.0)) if t % 5 else np.float32(s_in * 2.0 ** int(g.integers(-4, 5)))
        zp_in = int(g.integers(0, 256))
        x = np.arange(256, dtype=np.int32) if t % 2 else g.integers(-2 ** 31, 2 ** 31, size=200, dtype=np.int64).astype(np.int32)
        zi = zp_in if t % 2 else 0
        y = orc.requantize(x, [float(s_in)], zi, float(s_out), 0, "s32", "upward")
        ratio = Fraction(float(s_in)) / Fraction(float(s_out))
        pow2 = ratio.numerator & (ratio.numerator - 1) == 0 and ratio.denominator & (ratio.denominator - 1) == 0
        for xi, yi in zip(x.tolist(), y.tolist()):
            real = math.floor(ratio * (xi - zi) + Fraction(1, 2))
            real = max(-2 ** 31, min(2 ** 31 - 1, real))
            assert abs(yi - real) <= 1
            if pow2:
                assert yi == real


def test_requantize_fixed_differs_from_real_ratio_case(orc):
    # s_in = 1, s_out = 10: m = 0.1 -> (1717986918, -3); x = 5 gives fixed 0 but real 0.5 -> 1 (reading R4)
    assert orc.derive_multiplier(1.0 / 10.0) == (1717986918, -3)
    y = orc.requantize(np.array([5], np.int32), [1.0], 0, 10.0, 0, "s32", "upward")
    assert int(y[0]) == 0


def test_requantize_saturates(orc):
    x = np.array([-2 ** 31, -1000, 0, 1000, 2 ** 31 - 1], np.int32)
    y8 = orc.requantize(x, [1.0], 0, 1.0, 0, "s8")
    assert y8.tolist() == [-128, -128, 0, 127, 127]
    yu = orc.requantize(x, [1.0], 0, 1.0, 3, "u8")
    assert yu.tolist() == [0, 0, 3, 255, 255]


def test_zero_point_shift_u8_to_s8_lossless(orc):
    """Paper's VNNI legalize: u8 -> s8 with unchanged scale and zp-128 is
    an exact representation shift over all 256 codes."""
    q = np.arange(256, dtype=np.uint8)
    for zp in (0, 1, 77, 128, 200, 255):
        s = orc.requantize(q, [0.05], zp, 0.05, zp - 128, "s8")
        assert np.array_equal(s.astype(np.int64), q.astype(np.int64) - 128)
        # and the real values agree (Eq. 1)
        assert np.array_equal(s.astype(np.int64) - (zp - 128), q.astype(np.int64) - zp)


def test_requantize_per_channel_axis(orc):
    g = np.random.default_rng(4)
    x = g.integers(-5000, 5000, size=(3, 4, 5), dtype=np.int64).astype(np.int32)
    sc = np.array([0.5, 0.25, 0.125, 1.0], np.float32)
    y = orc.requantize(x, sc, 0, 1.0, 0, "s32", axis=1)
    for c in range(4):
        yc = orc.requantize(np.ascontiguousarray(x[:, c, :]), [sc[c]], 0, 1.0, 0, "s32")
        assert np.array_equal(y[:, c, :], yc)
