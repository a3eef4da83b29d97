"""GPU parity: standalone qnn.requantize / quantize / dequantize vs the oracle
(bit-exact integers; dequantize 0 ulp for 8-bit inputs, <= 1 ulp for int32)."""
import zlib

import numpy as np
import pytest
import torch

import oracle as orc
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    from paper_2006_10226_b200 import qnn
    qnn.lib()
    return qnn


def _rand(g, shape, dt):
    if dt == "s32":
        return g.integers(-2 ** 31, 2 ** 31, size=shape, dtype=np.int64).astype(np.int32)
    return gen.rand_q(g, shape, dt)


@pytest.mark.parametrize("in_dt", ["s32", "u8", "s8"])
@pytest.mark.parametrize("out_dt", ["u8", "s8", "s32"])
@pytest.mark.parametrize("mode", ["upward", "tonearest"])
def test_requantize_per_tensor(q, in_dt, out_dt, mode):
    g = np.random.default_rng(zlib.crc32(f"{in_dt}{out_dt}{mode}".encode()))
    for shape in [(1,), (17,), (3, 5, 7), (1000003,), (64, 56, 56, 3)]:
        x = _rand(g, shape, in_dt)
        zi = int(g.integers(-100, 100)) if in_dt != "u8" else int(g.integers(0, 256))
        if in_dt == "s8":
            zi = int(g.integers(-128, 128))
        s_in = float(np.float32(g.uniform(1e-4, 2.0)))
        s_out = float(np.float32(g.uniform(1e-3, 2.0) * (1000 if in_dt == "s32" else 1)))
        zo = 0 if out_dt == "s32" else int(g.integers(0, 256) if out_dt == "u8" else g.integers(-128, 128))
        want = orc.requantize(x, [s_in], zi, s_out, zo, out_dt, mode)
        got = q.qnn_requantize(torch.from_numpy(x).cuda(), [s_in], zi, s_out, zo, out_dt, mode).cpu().numpy()
        assert np.array_equal(got, want), (shape, np.argwhere(got != want)[:5])


@pytest.mark.parametrize("axis", [-1, 1])
def test_requantize_per_channel(q, axis):
    g = np.random.default_rng(7 + axis)
    x = _rand(g, (4, 96, 13, 40), "s32") if axis == 1 else _rand(g, (5, 7, 11, 1000), "s32")
    C = x.shape[axis]
    sc = g.uniform(1e-5, 1e-2, size=C).astype(np.float32)
    for mode in ("upward", "tonearest"):
        want = orc.requantize(x, sc, 3, 0.5, 100, "u8", mode, axis=axis)
        got = q.qnn_requantize(torch.from_numpy(x).cuda(), sc, 3, 0.5, 100, "u8", mode, axis=axis).cpu().numpy()
        assert np.array_equal(got, want)


def test_requantize_unaligned_views(q):
    g = np.random.default_rng(9)
    base = torch.from_numpy(_rand(g, (4099,), "u8")).cuda()
    for off in (1, 3, 15):
        x = base[off:off + 3001]
        want = orc.requantize(x.cpu().numpy(), [0.3], 7, 0.11, -5, "s8", "tonearest")
        got = q.qnn_requantize(x, [0.3], 7, 0.11, -5, "s8", "tonearest").cpu().numpy()
        assert np.array_equal(got, want)


def test_requantize_power_of_two_ties_separate_modes(q):
    """m = 0.5: odd inputs are exact ties; UPWARD and TONEAREST must differ on negatives."""
    x = np.arange(-1001, 1002, dtype=np.int32)
    up = q.qnn_requantize(torch.from_numpy(x).cuda(), [0.5], 0, 1.0, 0, "s32", "upward").cpu().numpy()
    tn = q.qnn_requantize(torch.from_numpy(x).cuda(), [0.5], 0, 1.0, 0, "s32", "tonearest").cpu().numpy()
    assert np.array_equal(up, orc.requantize(x, [0.5], 0, 1.0, 0, "s32", "upward"))
    assert np.array_equal(tn, orc.requantize(x, [0.5], 0, 1.0, 0, "s32", "tonearest"))
    assert (up != tn).sum() == 501


@pytest.mark.parametrize("out_dt", ["u8", "s8"])
def test_quantize(q, out_dt):
    g = np.random.default_rng(11)
    for shape, axis in [((100003,), -1), ((8, 3, 33, 17), 1), ((2, 224, 224, 3), -1)]:
        x = (g.standard_normal(shape) * 3).astype(np.float32)
        x.reshape(-1)[:4] = [np.nan, np.inf, -np.inf, 0.0]
        C = shape[axis] if shape[axis] <= 2048 else 1      # per-channel (<= 2048) or per-tensor
        sc = g.uniform(0.01, 0.1, size=C).astype(np.float32)
        zp = g.integers(0, 256, size=C) if out_dt == "u8" else g.integers(-128, 128, size=C)
        want = orc.quantize(x, sc, zp, out_dt, axis)
        got = q.qnn_quantize(torch.from_numpy(x).cuda(), sc, zp, out_dt, axis).cpu().numpy()
        assert np.array_equal(got, want)


@pytest.mark.parametrize("in_dt", ["u8", "s8", "s32"])
def test_dequantize(q, in_dt):
    g = np.random.default_rng(13)
    for shape, axis in [((100003,), -1), ((8, 3, 33, 17), 1)]:
        x = _rand(g, shape, in_dt)
        C = shape[axis] if shape[axis] <= 2048 else 1
        sc = g.uniform(1e-4, 0.1, size=C).astype(np.float32)
        zp = g.integers(0, 256, size=C) if in_dt == "u8" else g.integers(-128, 128, size=C)
        want = orc.dequantize(x, sc, zp, axis)
        got = q.qnn_dequantize(torch.from_numpy(x).cuda(), sc, zp, axis).cpu().numpy()
        if in_dt == "s32":
            # within 1 ulp of the single rounding (north_star tolerance)
            ulp = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
            assert ulp.max() <= 1
        else:
            assert np.array_equal(got.view(np.int32), want.view(np.int32))


def test_empty_tensor(q):
    x = torch.empty(0, dtype=torch.int32, device="cuda")
    y = q.qnn_requantize(x, [1.0], 0, 1.0, 0, "u8")
    assert y.numel() == 0


# ---- fast-path coverage: per-tensor int32 with zp_in == 0, and the two vectorised
# per-channel layouts (channel = fastest axis with C % 16 == 0; inner extent % 16 == 0)
FAST_LAYOUTS = [((3, 7, 9, 64), -1), ((2, 5, 11, 48), 3), ((4, 24, 8, 8), 1), ((2, 3, 16, 5), 1),
                ((2, 7, 3, 4), 1), ((5, 33, 129), 1)]


@pytest.mark.parametrize("in_dt", ["s32", "u8", "s8"])
@pytest.mark.parametrize("mode", ["upward", "tonearest"])
def test_requantize_fast_layouts(q, in_dt, mode):
    g = np.random.default_rng(zlib.crc32(f"fast{in_dt}{mode}".encode()))
    for shape, axis in FAST_LAYOUTS + [((40000,), -1)]:
        x = _rand(g, shape, in_dt)
        flat = x.reshape(-1)
        if in_dt == "s32":
            flat[:3] = [-2 ** 31, 2 ** 31 - 1, 0]
        C = shape[axis] if len(shape) > 1 else 1
        lo, hi = (1e-4, 1e-2) if in_dt == "s32" else (0.05, 2.0)
        sc = g.uniform(lo, hi, size=C).astype(np.float32)
        zi = 0 if in_dt == "s32" else int(g.integers(-128, 128) if in_dt == "s8" else g.integers(0, 256))
        for out_dt, zo in (("u8", 7), ("s8", -3), ("s32", 0)):
            want = orc.requantize(x, sc, zi, 0.7, zo, out_dt, mode, axis=axis)
            got = q.qnn_requantize(torch.from_numpy(x).cuda(), sc, zi, 0.7, zo, out_dt, mode,
                                   axis=axis).cpu().numpy()
            assert np.array_equal(got, want), (shape, axis, out_dt, np.argwhere(got != want)[:5])


@pytest.mark.parametrize("out_dt", ["u8", "s8"])
def test_quantize_fast_layouts(q, out_dt):
    g = np.random.default_rng(21)
    for shape, axis in FAST_LAYOUTS:
        x = (g.standard_normal(shape) * 3).astype(np.float32)
        x.reshape(-1)[:5] = [np.nan, np.inf, -np.inf, 0.0, 1e30]
        C = shape[axis]
        sc = g.uniform(0.01, 0.1, size=C).astype(np.float32)
        zp = g.integers(0, 256, size=C) if out_dt == "u8" else g.integers(-128, 128, size=C)
        want = orc.quantize(x, sc, zp, out_dt, axis)
        got = q.qnn_quantize(torch.from_numpy(x).cuda(), sc, zp, out_dt, axis).cpu().numpy()
        assert np.array_equal(got, want), (shape, axis)


@pytest.mark.parametrize("in_dt", ["u8", "s8"])
def test_dequantize_fast_layouts(q, in_dt):
    g = np.random.default_rng(23)
    for shape, axis in FAST_LAYOUTS:
        x = _rand(g, shape, in_dt)
        C = shape[axis]
        sc = g.uniform(1e-4, 0.1, size=C).astype(np.float32)
        zp = g.integers(0, 256, size=C) if in_dt == "u8" else g.integers(-128, 128, size=C)
        want = orc.dequantize(x, sc, zp, axis)
        got = q.qnn_dequantize(torch.from_numpy(x).cuda(), sc, zp, axis).cpu().numpy()
        assert np.array_equal(got.view(np.int32), want.view(np.int32)), (shape, axis)


def test_quantize_division_is_ieee_on_hard_cases(q):
    """The fast quantize divides via a Markstein-corrected reciprocal; it must equal the
    oracle's IEEE x / s on values that sit at or next to half-integers of x / s, and on
    awkward divisors (all-ones mantissas, powers of two, tiny/huge scales)."""
    g = np.random.default_rng(31)
    scales = np.array([np.float32(v) for v in (1.0, 0.5, 3.0, 0.1, 1 / 3, 0.0078125, 1e-30, 1e30)] +
                      [np.nextafter(np.float32(2.0), np.float32(0)), np.nextafter(np.float32(1.0), np.float32(0))] +
                      list(g.uniform(1e-3, 10, 6).astype(np.float32)), dtype=np.float32)
    for s in scales:
        k = np.arange(-300, 301, dtype=np.float64) + 0.5
        base = (k * np.float64(s)).astype(np.float32)
        near = np.concatenate([base, np.nextafter(base, np.float32(np.inf)), np.nextafter(base, np.float32(-np.inf)),
                               (g.standard_normal(200000) * 200 * np.float64(s)).astype(np.float32)])
        x = near.astype(np.float32)
        want = orc.quantize(x, [s], [128], "u8", -1)
        got = q.qnn_quantize(torch.from_numpy(x).cuda(), [float(s)], [128], "u8", -1).cpu().numpy()
        assert np.array_equal(got, want), (float(s), np.argwhere(got != want)[:5])
