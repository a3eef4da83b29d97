"""Oracle pins added in round 2 for the functions the round-1 review found unpinned:

* ``oracle.conv_multipliers`` (reading R3: m_k = (s_A * s_W[k]) / s_out in double, then R2's
  fixed-point form) against an independent derivation in exact rational arithmetic
  (``fractions.Fraction`` + ``math.frexp``), per-channel index included;
* the output clamp of ``oracle.requantize_acc`` (ReLU lower bound zp_out, TFLite-style
  act_min / act_max in the output domain, dtype saturation; readings R5 / R6) against
  hand-computed cases;
* ``oracle.dequantize`` of int32 input (Eq. 1, reading R14) against the exact rational
  value s * (q - zp): within one ulp everywhere, and correctly rounded when q - zp is exact
  in fp32.
"""
import math
from fractions import Fraction

import numpy as np
import pytest


def _derive_exact(m: float):
    """R2 restated from the definition: m = sig * 2^e, sig in [0.5, 1) (frexp is exact on a
    double); M = floor(sig * 2^31 + 1/2) (half away from zero, m > 0); carry renormalises."""
    sig, e = math.frexp(m)
    M = math.floor(Fraction(sig) * 2**31 + Fraction(1, 2))
    if M == 2**31:
        M, e = 2**30, e + 1
    return M, e


def test_conv_multipliers_vs_exact_rational(orc):
    g = np.random.default_rng(2024)
    checked = 0
    for trial in range(200):
        K = int(g.integers(1, 97))
        s_A = np.float32(10 ** g.uniform(-4, 0))
        s_out = np.float32(10 ** g.uniform(-3, 1))
        s_W = (10 ** g.uniform(-5, -1, size=K)).astype(np.float32)
        if trial % 7 == 0:
            s_W[: K // 2] = np.float32(2.0) ** -g.integers(3, 12, size=K // 2).astype(np.float32)   # dyadic ties
        M, S = orc.conv_multipliers(float(s_A), s_W, float(s_out), K)
        for k in range(K):
            # R3: the fp32 product is exact in double; ONE correctly rounded division
            m = float(Fraction(float(s_A)) * Fraction(float(s_W[k])) / Fraction(float(s_out)))
            Mk, ek = _derive_exact(m)
            assert (int(M[k]), int(S[k])) == (Mk, ek), (trial, k)
            checked += 1
    # per-tensor: one scale broadcast to every channel
    M, S = orc.conv_multipliers(0.02, [0.003], 0.5, 5)
    Mk, ek = _derive_exact(float(Fraction(float(np.float32(0.02))) * Fraction(float(np.float32(0.003)))
                                 / Fraction(float(np.float32(0.5)))))
    assert all(int(M[k]) == Mk and int(S[k]) == ek for k in range(5))
    assert checked > 9000


def test_conv_multipliers_product_rounded_once(orc):
    """A triple where rounding the product to fp32 first (a common shortcut) changes M:
    the oracle must follow R3 (exact product, one division)."""
    g = np.random.default_rng(5)
    found = 0
    for _ in range(20000):
        a, w, o = (np.float32(x) for x in 10 ** g.uniform(-3, 0, size=3))
        exact = float(Fraction(float(a)) * Fraction(float(w)) / Fraction(float(o)))
        shortcut = float(np.float32(a * w)) / float(o)
        if _derive_exact(exact) != _derive_exact(shortcut):
            M, S = orc.conv_multipliers(float(a), [w], float(o), 1)
            assert (int(M[0]), int(S[0])) == _derive_exact(exact)
            found += 1
            if found >= 20:
                break
    assert found >= 5


# m = 1 exactly (M = 2^30, shift 1): R(acc) = acc, so every output below is hand-computable
_CLAMP_CASES = [
    # dtype, zp_out, relu, act_min, act_max, acc, expected
    ("s8", -10, False, -5, 20, [-200, -6, 4, 5, 25, 30, 31, 200], [-5, -5, -5, -5, 15, 20, 20, 20]),
    ("s8", -10, True, -5, 20, [-200, -6, 4, 5, 25, 30, 31, 200], [-5, -5, -5, -5, 15, 20, 20, 20]),
    ("s8", -10, True, None, None, [-200, -6, 4, 5, 25, 30, 31, 200], [-10, -10, -6, -5, 15, 20, 21, 127]),
    ("s8", 7, False, None, None, [-300, -135, -134, 0, 120, 121, 500], [-128, -128, -127, 7, 127, 127, 127]),
    # MobileNet-style ReLU6 as an output-domain clamp: act_max = zp_out + round(6 / s_out)
    ("u8", 3, True, None, 63, [-5, 0, 10, 59, 60, 61, 300], [3, 3, 13, 62, 63, 63, 63]),
    ("u8", 3, False, 1, 63, [-5, -2, -1, 0, 61], [1, 1, 2, 3, 63]),
    ("u8", 0, False, None, None, [-1, 0, 255, 256], [0, 0, 255, 255]),
]


@pytest.mark.parametrize("dt,zp,relu,amin,amax,acc,want", _CLAMP_CASES)
def test_requantize_output_clamp_hand_cases(orc, dt, zp, relu, amin, amax, acc, want):
    M, shift = orc.derive_multiplier(1.0)
    assert (M, shift) == (2**30, 1)
    for mode in ("upward", "tonearest"):
        y = orc.requantize_acc(np.array(acc, np.int64)[None, :], [M], [shift], dt, zp, mode, relu, amin, amax,
                               axis=0)
        assert y[0].tolist() == want, mode


def test_requantize_output_clamp_with_rounding(orc):
    """m = 1/2 (M = 2^30, shift 0): rounding happens before the clamp (R5)."""
    M, shift = orc.derive_multiplier(0.5)
    acc = np.array([[3, 4, 5, 6, -3, -4]], np.int64)
    up = orc.requantize_acc(acc, [M], [shift], "s8", 0, "upward", False, None, 2, axis=0)[0].tolist()
    assert up == [2, 2, 2, 2, -1, -2]                     # 1.5 -> 2, 2.5 -> 3 -> 2, -1.5 -> -1
    tn = orc.requantize_acc(acc, [M], [shift], "s8", 0, "tonearest", True, None, 2, axis=0)[0].tolist()
    assert tn == [2, 2, 2, 2, 0, 0]                       # ReLU: lower bound zp_out = 0


def test_dequantize_int32_vs_exact(orc):
    g = np.random.default_rng(17)
    q = g.integers(-2**31, 2**31, size=20000).astype(np.int32)
    q[:6] = [2**31 - 1, -2**31, 0, 1, -1, 2**24 + 1]
    for zp, s in ((0, np.float32(0.0123)), (-2**31, np.float32(3.5e-7)), (12345, np.float32(1.7)),
                  (2**31 - 1, np.float32(2.0**-20))):
        x = orc.dequantize(q, [s], [zp])
        for qi, xi in zip(q.tolist(), x.tolist()):
            v = Fraction(float(s)) * (qi - zp)
            ulp = Fraction(float(np.spacing(np.float32(abs(xi)))))
            assert abs(Fraction(xi) - v) <= ulp, (qi, zp, float(s))
            if abs(qi - zp) <= 2**24:           # q - zp exact in fp32: a single rounding
                assert xi == float(np.float32(float(v))) or abs(Fraction(xi) - v) <= ulp / 2


@pytest.mark.parametrize("groups", [1, 6])
def test_per_channel_weight_zero_points_vs_float64_library(orc, groups):
    """f4 (per-channel zp_W): the oracle's channel-by-channel evaluation against torch's float64
    conv of the zero-point-subtracted operands (exact below 2^53), with W - zp_W[k] broadcast."""
    import torch
    import torch.nn.functional as F
    g = np.random.default_rng(31 + groups)
    for trial in range(6):
        C = 6
        K = 6 if groups > 1 else int(g.integers(2, 9))
        A = g.integers(0, 256, size=(2, C, 7, 8)).astype(np.uint8)
        Wt = g.integers(-128, 128, size=(K, C // groups, 3, 3)).astype(np.int8)
        zpA = int(g.integers(0, 256))
        zpv = g.integers(-127, 128, size=K).astype(np.int32)
        bias = g.integers(-999, 1000, size=K).astype(np.int32)
        got = orc.conv2d_acc(A, Wt, zpA, zpv, bias, (1, 2), (1, 1, 0, 2), (1, 1), groups)
        a = F.pad(torch.from_numpy(A.astype(np.float64) - zpA), (1, 2, 1, 0))
        w = torch.from_numpy(Wt.astype(np.float64) - zpv.astype(np.float64)[:, None, None, None])
        want = F.conv2d(a, w, stride=(1, 2), groups=groups).numpy().astype(np.int64) + bias[None, :, None, None]
        assert np.array_equal(got, want), trial
    Ad = g.integers(0, 256, size=(5, 40)).astype(np.uint8)
    Wd = g.integers(0, 256, size=(7, 40)).astype(np.uint8)
    zd = g.integers(0, 256, size=7)
    got = orc.dense_acc(Ad, Wd, 17, zd)
    want = (Ad.astype(np.int64) - 17) @ (Wd.astype(np.int64) - zd[:, None]).T
    assert np.array_equal(got, want)
