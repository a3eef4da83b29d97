"""Pins for the oracle's inter-layer glue: qnn.add, max / average
pooling and the conv + residual-add composition.  Each check ties the oracle to
something other than itself: SPEC's worked examples (canonicalize_add / *_pool), exact
rational arithmetic on small inputs, brute-force sliding windows in numpy, algebraic
reductions to already-pinned operators."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as orc
from workloads import gen


# ----------------------------------------------------------------------------- qnn.add
def test_add_spec_examples():
    # SPEC canonicalize_add: lhs 1.0 and rhs 1.0 under scale 0.5 / zp 0 in and out -> 4 (represents 2.0)
    one = np.array([2], np.uint8)
    assert orc.add(one, 0.5, 0, one, 0.5, 0, 0.5, 0, "u8").tolist() == [4]
    # identical params, zp 0 -> clamp(Q_L + Q_R)
    g = np.random.default_rng(1)
    a = g.integers(-128, 128, 5000).astype(np.int8)
    b = g.integers(-128, 128, 5000).astype(np.int8)
    want = np.clip(a.astype(np.int64) + b, -128, 127)
    assert np.array_equal(orc.add(a, 0.37, 0, b, 0.37, 0, 0.37, 0, "s8"), want)
    # saturation: s8 output, values summing beyond 127 -> 127
    assert orc.add(np.array([100], np.int8), 1.0, 0, np.array([100], np.int8), 1.0, 0, 1.0, 0, "s8").tolist() == [127]


def _round_half_away(fr: Fraction) -> int:
    a = abs(fr)
    m = (a.numerator * 2 + a.denominator) // (2 * a.denominator)
    return m if fr >= 0 else -m


@pytest.mark.parametrize("mode", ["upward", "tonearest"])
def test_add_matches_real_sum_within_two_roundings(mode):
    """Each input is rounded once (Eq. 5), so the result is within 1 of the real sum
    rounded once (two half-ulp errors); zero error when both ratios are powers of two."""
    g = np.random.default_rng(2)
    for _ in range(20):
        s_a, s_b, s_o = (float(np.float32(v)) for v in g.uniform(0.01, 0.2, 3))
        za, zb, zo = (int(v) for v in g.integers(0, 256, 3))
        a = g.integers(0, 256, 400).astype(np.uint8)
        b = g.integers(0, 256, 400).astype(np.uint8)
        got = orc.add(a, s_a, za, b, s_b, zb, s_o, zo, "s32", mode).astype(np.int64)
        for i in range(a.size):
            real = (Fraction(s_a) * (int(a[i]) - za) + Fraction(s_b) * (int(b[i]) - zb)) / Fraction(s_o)
            assert abs(got[i] - (_round_half_away(real) + zo)) <= 1
    a = g.integers(0, 256, 1000).astype(np.uint8)
    b = g.integers(0, 256, 1000).astype(np.uint8)
    got = orc.add(a, 0.25, 7, b, 0.5, 3, 0.5, 11, "s32", mode).astype(np.int64)
    ya = np.array([_round_half_away(Fraction(int(v) - 7, 2)) if mode == "tonearest" else
                   int(np.floor(Fraction(int(v) - 7, 2) + Fraction(1, 2))) for v in a])
    assert np.array_equal(got, ya + (b.astype(np.int64) - 3) + 11)


def test_add_is_commutative_and_relu_bounded():
    g = np.random.default_rng(3)
    a = g.integers(0, 256, 3000).astype(np.uint8)
    b = g.integers(-128, 128, 3000).astype(np.int8)
    x = orc.add(a, 0.031, 120, b, 0.017, -3, 0.05, 9, "u8", "upward", relu=True)
    y = orc.add(b, 0.017, -3, a, 0.031, 120, 0.05, 9, "u8", "upward", relu=True)
    assert np.array_equal(x, y)
    assert x.min() >= 9


# ----------------------------------------------------------------------------- pooling
def test_pool_spec_examples():
    x = np.array([[[[1, 2], [3, 4]]]], np.uint8)
    assert orc.pool2d(x, "avg", 2, 2, (2, 2)).item() == 3          # round(2.5) = 3, ties away
    assert orc.pool2d(x, "max", 2, 2, (2, 2)).item() == 4
    v = np.full((1, 2, 5, 5), 77, np.uint8)
    assert (orc.pool2d(v, "avg", 3, 3, (1, 1), (1, 1, 1, 1)) == 77).all()   # average of equals
    w = np.full((1, 1, 3, 3), 255, np.uint8)
    assert orc.pool2d(w, "avg", 3, 3).item() == 255                 # 2295 / 9, no overflow
    n = np.array([[[[-1, -2], [-2, -1]]]], np.int8)                  # -1.5 -> -2 (away from zero)
    assert orc.pool2d(n, "avg", 2, 2, (2, 2)).item() == -2


def _windows(x, R, S, stride, pad):
    N, C, H, W = x.shape
    P, Q = orc.out_hw(H, W, R, S, stride, pad)
    for p in range(P):
        for q in range(Q):
            hs = [p * stride[0] + r - pad[0] for r in range(R)]
            ws = [q * stride[1] + s - pad[1] for s in range(S)]
            hs = [h for h in hs if 0 <= h < H]
            ws = [w for w in ws if 0 <= w < W]
            yield p, q, x[:, :, hs][:, :, :, ws]


@pytest.mark.parametrize("dt", ["u8", "s8"])
@pytest.mark.parametrize("cfg", [(3, 3, (2, 2), (1, 1, 1, 1)), (2, 2, (2, 2), (0, 0, 0, 0)),
                                 (3, 2, (1, 2), (1, 0, 1, 1)), (7, 7, (1, 1), (0, 0, 0, 0))])
def test_pool_brute_force(dt, cfg):
    R, S, st, pad = cfg
    g = np.random.default_rng(4)
    x = gen.rand_q(g, (2, 3, 9, 8) if R < 7 else (2, 3, 7, 7), dt)
    mx = orc.pool2d(x, "max", R, S, st, pad)
    av = orc.pool2d(x, "avg", R, S, st, pad)
    for p, q, win in _windows(x, R, S, st, pad):
        w = win.reshape(win.shape[0], win.shape[1], -1).astype(np.int64)
        assert np.array_equal(mx[:, :, p, q], w.max(axis=2))
        for n in range(w.shape[0]):
            for c in range(w.shape[1]):
                assert av[n, c, p, q] == _round_half_away(Fraction(int(w[n, c].sum()), w.shape[2]))


# ----------------------------------------------------------------------------- conv + residual
def test_conv_add_reduces_to_conv_for_a_zero_residual():
    case = gen.conv_case(41, 2, 16, 9, 9, 24, 3, 3, (1, 1), (1, 1, 1, 1))
    res = np.full((2, 24, 9, 9), 37, np.uint8)                      # residual == its zero point
    got = orc.qnn_conv2d_add(case.nchw(), case.oihw(), case.zp_A, case.zp_W, case.s_A, case.s_W, case.bias,
                             res, 0.02, 37, case.out_params(), case.stride, case.pad)
    want = orc.qnn_conv2d(case.nchw(), case.oihw(), case.zp_A, case.zp_W, case.s_A, case.s_W, case.bias,
                          case.out_params(), case.stride, case.pad)
    assert np.array_equal(got, want)


def test_conv_add_reduces_to_requantize_for_a_zero_conv():
    case = gen.conv_case(42, 1, 8, 6, 6, 8, 1, 1, bias=False)
    Wz = np.zeros_like(case.oihw())
    g = np.random.default_rng(5)
    res = g.integers(0, 256, (1, 8, 6, 6)).astype(np.uint8)
    out = dict(case.out_params(), relu=False, act_min=None, act_max=None)
    got = orc.qnn_conv2d_add(case.nchw(), Wz, case.zp_A, 0, case.s_A, case.s_W, None, res, 0.03, 100, out)
    want = orc.requantize(res, [0.03], 100, out["scale"], out["zero_point"], out["dtype"], out["rounding"])
    assert np.array_equal(got, want)
