"""Oracle pins: quantize / dequantize (Eq. 1; reading R14)."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["quantize"], ids=lambda e: str(e["x"]))
def test_quantize_spec_examples(orc, ex):
    q = orc.quantize(np.array([ex["x"]], np.float32), [ex["scale"]], [ex["zp"]], ex["dtype"])
    assert int(q[0]) == ex["q"]


@pytest.mark.parametrize("ex", GOLD["dequantize"], ids=lambda e: str(e["q"]))
def test_dequantize_spec_examples(orc, ex):
    x = orc.dequantize(np.array([ex["q"]], np.uint8), [ex["scale"]], [ex["zp"]])
    assert float(x[0]) == ex["x"]


def test_quantize_vs_exact_rational():
    """Against Fraction(x)/Fraction(s) rounded half away from zero: the fp32
    quotient may move a value across a .5 boundary only when it lies within one
    ulp of that boundary (reading R14)."""
    import oracle as orc
    g = np.random.default_rng(41)
    x = (g.standard_normal(20000) * 40).astype(np.float32)
    x[:100] = (np.arange(100, dtype=np.float32) - 50) * np.float32(0.5) * np.float32(0.1)   # near-ties
    s = np.float32(0.1)
    q = orc.quantize(x, [s], [3], "s8").astype(np.int64)
    for xi, qi in zip(x.tolist(), q.tolist()):
        r = Fraction(xi) / Fraction(float(s))
        fl = math.floor(abs(r) + Fraction(1, 2))
        exact = (fl if r >= 0 else -fl) + 3
        exact = max(-128, min(127, exact))
        if exact != qi:
            t = float(np.float32(xi) / s)
            ulp = np.spacing(np.float32(abs(t)))
            frac = abs(r) - math.floor(abs(r))
            assert abs(qi - exact) == 1
            assert abs(frac - Fraction(1, 2)) <= Fraction(float(ulp)), (xi, qi, exact)


def test_quantize_fp32_division_semantics(orc):
    """Bit-level: q == clamp(round_half_away(np.float32(x)/np.float32(s)) + zp) (IEEE fp32 division, numpy)."""
    g = np.random.default_rng(42)
    x = (g.standard_normal(50000) * 100).astype(np.float32)
    for s, zp, dt in [(np.float32(0.37), 128, "u8"), (np.float32(1.7), -5, "s8")]:
        q = orc.quantize(x, [s], [zp], dt).astype(np.int64)
        t = (x / s).astype(np.float32)
        r = np.where(t >= 0, np.floor(np.abs(t).astype(np.float64) + 0.5), -np.floor(np.abs(t).astype(np.float64) + 0.5))
        lo, hi = (0, 255) if dt == "u8" else (-128, 127)
        assert np.array_equal(q, np.clip(r.astype(np.int64) + zp, lo, hi))


def test_quantize_special_values(orc):
    x = np.array([np.nan, np.inf, -np.inf, 1e30, -1e30, 0.0, -0.0], np.float32)
    q = orc.quantize(x, [0.5], [7], "u8")
    assert q.tolist() == [7, 255, 0, 255, 0, 7, 7]


def test_dequantize_single_rounding(orc):
    """fl32(s*(q-zp)) with one rounding: compare with numpy float64 product then
    float32 cast (exact in float64 for 8-bit q; library pin)."""
    g = np.random.default_rng(43)
    for dt, lo, hi in [("u8", 0, 255), ("s8", -128, 127)]:
        q = g.integers(lo, hi + 1, size=4096).astype(np.uint8 if dt == "u8" else np.int8)
        for s in (np.float32(0.0123), np.float32(3.3e-5), np.float32(17.25)):
            zp = int(g.integers(lo, hi + 1))
            got = orc.dequantize(q, [s], [zp])
            ref = ((q.astype(np.float64) - zp) * np.float64(s)).astype(np.float32)
            assert np.array_equal(got.view(np.int32), ref.view(np.int32))


def test_dequant_of_quant_within_half_scale(orc):
    """|dequantize(quantize(x)) - x| <= s/2 for x inside the representable range."""
    g = np.random.default_rng(44)
    s, zp = np.float32(0.05), 100
    lo, hi = (0 - zp) * float(s), (255 - zp) * float(s)
    x = g.uniform(lo, hi, size=20000).astype(np.float32)
    y = orc.dequantize(orc.quantize(x, [s], [zp], "u8"), [s], [zp])
    assert np.all(np.abs(y.astype(np.float64) - x.astype(np.float64)) <= float(s) / 2 * (1 + 1e-6))


def test_per_channel_params(orc):
    g = np.random.default_rng(45)
    x = g.standard_normal((2, 3, 4)).astype(np.float32)
    sc = np.array([0.1, 0.2, 0.3], np.float32)
    zp = np.array([1, 2, 3], np.int32)
    q = orc.quantize(x, sc, zp, "s8", axis=1)
    for c in range(3):
        assert np.array_equal(q[:, c], orc.quantize(np.ascontiguousarray(x[:, c]), [sc[c]], [zp[c]], "s8"))
    d = orc.dequantize(q, sc, zp, axis=1)
    for c in range(3):
        assert np.array_equal(d[:, c], orc.dequantize(np.ascontiguousarray(q[:, c]), [sc[c]], [zp[c]]))
