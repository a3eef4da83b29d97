"""GPU parity on edge cases of the kernels' fast paths (round-2 review items), bit-exact
against the oracle on seeded inputs:

* 3x3 depthwise through the TMA-staged kernel with column padding >= 2 (the middle tap
  can fall outside the image; TMA's zero fill is not zp_A);
* standalone requantize of int32 input with zp_in != 0 at right shift 63 (reading R15:
  |x - zp_in| reaches 2^32 - 1, so x * M reaches [2^62, 2^63) and rounds to +-1);
* the channel-major pointwise GEMM with folded offsets near +-2^30 (the 64-bit K of the
  fast requantize) and on its generic path (TONEAREST), and the weight code -128;
* the pixel-major GEMM's generic rounding path forced by a multiplier outside the fast
  shift range, with large biases.
"""
import numpy as np
import pytest
import torch

import oracle as orc
from gpu_helpers import gpu_conv, mismatch_report, oracle_conv
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pad", [(2, 2, 2, 2), (1, 1, 2, 2), (0, 2, 0, 2), (2, 0, 2, 0), (3, 3, 3, 3)])
@pytest.mark.parametrize("stride", [1, 2])
@pytest.mark.parametrize("C", [32, 48])
def test_depthwise_tma_wide_padding(pad, stride, C):
    """u8 input with zp_A = 128: every out-of-image tap must contribute (zp_A - zp_A) = 0."""
    for mode in ("upward", "tonearest"):
        case = gen.conv_case(7100 + C + 7 * stride + sum(pad), 2, C, 9, 10, C, 3, 3, (stride, stride), pad, (1, 1), C,
                             "u8", "s8", zp_A=128, relu=False, rounding=mode)
        _, _, y = gpu_conv(case)
        got, want = y.cpu().numpy(), oracle_conv(case)
        assert got.shape == want.shape
        assert np.array_equal(got, want), f"pad {pad} stride {stride} {mode}\n" + mismatch_report(got, want)


def test_depthwise_tma_narrow_image_padding():
    """W = 2 with pad 2: some output columns see no in-image tap at all."""
    case = gen.conv_case(7190, 1, 16, 5, 2, 16, 3, 3, (1, 1), (2, 2, 2, 2), (1, 1), 16, "u8", "s8", zp_A=200,
                         relu=False)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), mismatch_report(got, want)


@pytest.mark.parametrize("mode", ["upward", "tonearest"])
@pytest.mark.parametrize("out_dtype", ["s8", "u8", "s32"])
def test_requantize_int32_shift63(mode, out_dtype):
    """m in [2^-33, 2^-32) gives right shift 63.  With zp_in = INT32_MIN, x - zp_in spans
    [0, 2^32 - 1] and the exact result is 0 or 1 (UPWARD) -- previously flushed to 0."""
    from paper_2006_10226_b200 import qnn_requantize
    g = np.random.default_rng(8)
    x = np.concatenate([np.array([2**31 - 1, 2**31 - 2, -2**31, 0, 2**30, -1], np.int64),
                        g.integers(-2**31, 2**31, size=4090)]).astype(np.int32)
    for zp_in in (-2**31, 2**31 - 1, -12345):
        for s_out in (1.5 * 2.0**32, 1.999 * 2.0**32, 2.0**33 - 2.0**10, 1.0000001 * 2.0**32):
            s_out = float(np.float32(s_out))
            zp_out = 0 if out_dtype != "u8" else 3
            got = qnn_requantize(torch.from_numpy(x).cuda(), [1.0], zp_in, s_out, zp_out, out_dtype, mode).cpu().numpy()
            want = orc.requantize(x, [1.0], zp_in, s_out, zp_out, out_dtype, mode)
            assert np.array_equal(got, want), f"zp_in {zp_in} s_out {s_out}\n" + mismatch_report(got, want)
            if zp_in == -2**31:
                assert (want.astype(np.int64) - zp_out).max() >= 1   # the case is really reached


@pytest.mark.parametrize("mode", ["upward", "tonearest"])
@pytest.mark.parametrize("K", [128, 256])
def test_channel_major_large_offsets(mode, K):
    """1x1 convs on the channel-major kernel with biases near +-2^30: the folded offset
    dominates, and the fast path's 64-bit K = off * M + c must stay exact."""
    g = np.random.default_rng(61 + K)
    N, H, W, C = 2, 13, 11, 128
    A = gen.rand_q(g, (N, H, W, C), "u8")
    Wt = gen.rand_q(g, (K, 1, 1, C), "s8")           # full range, -128 included
    bias = (np.where(g.random(K) < 0.5, -1, 1) * g.integers(2**29, 2**30, size=K)).astype(np.int32)
    s_A = 0.02
    s_W = g.uniform(0.002, 0.02, size=K).astype(np.float32)
    # output scale sized to the bias magnitude so outputs stay inside u8 for most channels
    s_out = float(np.float32(2.0**31 * s_A * float(np.median(s_W)) / 200.0))
    case = gen.ConvCase(A, Wt, bias, 117, 0, s_A, s_W, s_out, 128, "u8", (1, 1), (0, 0, 0, 0), (1, 1), 1, False,
                        None, None, mode)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), mismatch_report(got, want)
    assert len(np.unique(want)) > 50                 # not saturated


@pytest.mark.parametrize("mode", ["upward", "tonearest"])
def test_weights_code_minus128(mode):
    """Every weight -128 (the s8 extreme, zp_W = 0) on the pixel-major, channel-major and
    depthwise kernels."""
    for (C, K, R, groups, pad) in ((64, 64, 3, 1, 1), (64, 256, 1, 1, 0), (32, 32, 3, 32, 1)):
        case = gen.conv_case(7300 + K + R, 2, C, 10, 9, K, R, R, (1, 1), (pad,) * 4, (1, 1), groups, "u8", "s8",
                             rounding=mode, relu=False)
        case.W[...] = -128
        case.s_out = float(np.float32(case.s_out * 4))
        _, _, y = gpu_conv(case)
        got, want = y.cpu().numpy(), oracle_conv(case)
        assert np.array_equal(got, want), f"C{C} K{K} R{R} g{groups}\n" + mismatch_report(got, want)


@pytest.mark.parametrize("mode", ["upward", "tonearest"])
def test_pixel_major_generic_path_large_bias(mode):
    """m = 200 / 2^31 gives right shift 54 (outside the fast range [33, 52]): the 64-bit
    generic rounding on the pixel-major kernel, with biases near 2^30 and 3x3 border classes;
    channel 5 (m ~ 2^-11.4, shift 42) is a fast-range channel in the same tiles."""
    g = np.random.default_rng(71)
    N, H, W, C, K = 2, 12, 12, 32, 96
    A = gen.rand_q(g, (N, H, W, C), "u8")
    Wt = gen.rand_q(g, (K, 3, 3, C), "s8")
    bias = g.integers(-2**30, 2**30, size=K).astype(np.int32)
    s_A = 0.5
    s_W = np.full(K, 2.0**-12, np.float32)
    s_W[5] = 1.0
    s_out = float(np.float32(2.0**31 * s_A * 2.0**-12 / 200.0))
    case = gen.ConvCase(A, Wt, bias, 90, 0, s_A, s_W, s_out, 128, "u8", (1, 1), (1, 1, 1, 1), (1, 1), 1, False,
                        None, None, mode)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), mismatch_report(got, want)


def _guarded(shape, dtype, guard=4096, fill=0xA5):
    """An output view inside a larger buffer whose guard bytes (before, after) hold `fill`."""
    n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
    raw = torch.full((guard + n + guard,), fill, dtype=torch.uint8, device="cuda")
    view = raw[guard:guard + n].view(dtype).view(shape)
    return raw, view


@pytest.mark.parametrize("kind", ["pointwise_t", "rows3x3", "stem_build", "im2col", "depthwise", "dense_raw",
                                  "channel_slice"])
def test_no_writes_outside_the_output(kind):
    """compute-sanitizer is closed on this pool, so out-of-bounds WRITES are checked directly:
    every kernel family writes into a view of a buffer with 4 KB guard zones on both sides (and,
    for a channel-strided output, into every other channel slice), which must stay untouched."""
    from paper_2006_10226_b200 import PackedConv2d, PackedDense
    from gpu_helpers import to_dev
    cases = {
        "pointwise_t": gen.conv_case(7401, 2, 64, 9, 7, 256, 1, 1),
        "rows3x3": gen.conv_case(7402, 1, 64, 11, 9, 64, 3, 3, (1, 1), (1, 1, 1, 1)),
        "stem_build": gen.conv_case(7403, 2, 3, 30, 30, 64, 7, 7, (2, 2), (3, 3, 3, 3)),
        "im2col": gen.conv_case(7404, 2, 96, 9, 9, 130, 3, 3, (2, 2), (1, 1, 1, 1)),
        "depthwise": gen.conv_case(7405, 2, 48, 9, 10, 48, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), 48),
        "channel_slice": gen.conv_case(7406, 2, 64, 8, 8, 128, 1, 1),
    }
    if kind == "dense_raw":
        d = gen.dense_case(7407, 100, 300, 512, out_dtype="s32")
        op = PackedDense(100, to_dev(d.W), to_dev(d.bias), d.zp_A, d.zp_W, d.s_A, d.s_W, None)
        raw, y = _guarded((100, 300), torch.int32)
        op(to_dev(d.A), out=y)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), orc.qnn_dense(d.A, d.W, d.zp_A, d.zp_W, d.s_A, d.s_W, d.bias, None))
    else:
        c = cases[kind]
        N, H, W, C = c.A.shape
        wide = kind == "channel_slice"
        K = c.W.shape[0]
        op = PackedConv2d(N, H, W, C, to_dev(c.W), to_dev(c.bias), c.zp_A, c.zp_W, c.s_A, c.s_W, c.out_params(),
                          c.stride, c.pad, c.dil, c.groups, out_cstride=3 * K if wide else 0)
        oshape = op.out_shape()
        raw, y = _guarded(oshape, torch.uint8)
        if wide:
            op(to_dev(c.A), out=y, out_channel_offset=K)
        else:
            op(to_dev(c.A), out=y)
        torch.cuda.synchronize()
        got = y.cpu().numpy()
        want = oracle_conv(c)
        if wide:
            assert np.array_equal(got[..., K:2 * K], want)
            assert (got[..., :K] == 0xA5).all() and (got[..., 2 * K:] == 0xA5).all()
        else:
            assert np.array_equal(got, want)
    r = raw.cpu().numpy()
    assert (r[:4096] == 0xA5).all() and (r[-4096:] == 0xA5).all(), "write outside the output"
