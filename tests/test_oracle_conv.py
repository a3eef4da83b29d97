"""Oracle pins: quantized conv2d / dense (Eq. 2, Eq. 3, zero-point padding P:259).

Pins that do not reuse the oracle's own formula:
  * SPEC scalar example and a hand-derived 1-D zero-point padding case;
  * PyTorch's float64 conv2d / numpy int64 matmul on the zp-subtracted
    operands — exact here since |sum| < 2^53 (library routine, independent);
  * the Eq. 2 == Eq. 3 identity on brute-force tiny shapes;
  * invariants: zp shift invariance, explicit zp pre-padding, depthwise ==
    per-channel convs, dense == 1x1 conv, saturation, ReLU commutation.
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from workloads import gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _torch_ref(A, W, zpA, zpW, bias, stride, pad, dil, groups):
    """sum (A - zpA)(W - zpW) via torch float64 conv; zero padding in the
    subtracted domain == zp_A padding in the quantized domain."""
    a = torch.from_numpy(A.astype(np.float64) - zpA)
    w = torch.from_numpy(W.astype(np.float64) - zpW)
    pt, pl, pb, pr = pad
    a = F.pad(a, (pl, pr, pt, pb))
    out = F.conv2d(a, w, None, stride, 0, dil, groups)
    r = out.numpy()
    assert np.all(np.abs(r) < 2 ** 52)
    r = r.astype(np.int64)
    if bias is not None:
        r += bias.reshape(1, -1, 1, 1).astype(np.int64)
    return r


def test_conv_scalar_spec_example(orc):
    ex = GOLD["conv_scalar"][0]
    A = np.array([[[[ex["qa"]]]]], np.uint8)
    W = np.array([[[[ex["qw"]]]]], np.uint8)
    assert orc.conv2d_acc(A, W, ex["zp_a"], ex["zp_w"])[0, 0, 0, 0] == ex["acc"]
    assert orc.conv2d_eq3(A, W, ex["zp_a"], ex["zp_w"])[0, 0, 0, 0] == ex["acc"]
    assert orc.dense_acc(A.reshape(1, 1), W.reshape(1, 1), ex["zp_a"], ex["zp_w"])[0, 0] == ex["acc"]


def test_conv_zero_point_padding_1d(orc):
    """row [10, 20], zp_A = 10, W = [1, 2, 3], zp_W = 0, pad 1:
    padded row [10, 10, 20, 10] - 10 = [0, 0, 10, 0] -> [0+0+30, 0+20+0] = [30, 20].
    Naive zero padding would give [20, -10]."""
    A = np.array([10, 20], np.uint8).reshape(1, 1, 1, 2)
    W = np.array([1, 2, 3], np.int8).reshape(1, 1, 1, 3)
    out = orc.conv2d_acc(A, W, 10, 0, pad=(0, 1, 0, 1))
    assert out.reshape(-1).tolist() == [30, 20]


def _rand_shape(g):
    groups = int(g.choice([1, 1, 2, 0]))
    C = int(g.integers(1, 5))
    if groups == 0:           # depthwise
        groups = C
        K = C * int(g.integers(1, 3))
    else:
        C *= groups
        K = groups * int(g.integers(1, 4))
    H, W = int(g.integers(1, 9)), int(g.integers(1, 9))
    R, S = int(g.integers(1, 4)), int(g.integers(1, 4))
    st = (int(g.integers(1, 3)), int(g.integers(1, 3)))
    dil = (int(g.integers(1, 3)), int(g.integers(1, 3)))
    pad = tuple(int(v) for v in g.integers(0, 3, size=4))
    if H + pad[0] + pad[2] < dil[0] * (R - 1) + 1 or W + pad[1] + pad[3] < dil[1] * (S - 1) + 1:
        pad = (R * dil[0], S * dil[1], R * dil[0], S * dil[1])
    return dict(N=int(g.integers(1, 3)), C=C, H=H, W=W, K=K, R=R, S=S, stride=st, pad=pad, dil=dil, groups=groups)


ZPS = {"u8": [0, 1, 127, 128, 255], "s8": [-128, -1, 0, 1, 127]}


@pytest.mark.parametrize("adt,wdt", [("u8", "s8"), ("u8", "u8"), ("s8", "s8"), ("s8", "u8")])
def test_conv_matches_torch_float64(orc, adt, wdt):
    """Direct form vs a library conv on zp-subtracted operands, 125 S:607-style draws per dtype pair."""
    g = np.random.default_rng({"u8s8": 11, "u8u8": 12, "s8s8": 13, "s8u8": 14}[adt + wdt])
    for i in range(125):
        sh = _rand_shape(g)
        A = gen.rand_q(g, (sh["N"], sh["C"], sh["H"], sh["W"]), adt)
        W = gen.rand_q(g, (sh["K"], sh["C"] // sh["groups"], sh["R"], sh["S"]), wdt)
        zpA = int(g.choice(ZPS[adt]))
        zpW = int(g.choice(ZPS[wdt]))
        bias = g.integers(-1000, 1000, size=sh["K"]).astype(np.int32) if i % 2 else None
        kw = dict(stride=sh["stride"], pad=sh["pad"], dil=sh["dil"], groups=sh["groups"])
        got = orc.conv2d_acc(A, W, zpA, zpW, bias, **kw)
        ref = _torch_ref(A, W, zpA, zpW, bias, sh["stride"], sh["pad"], sh["dil"], sh["groups"])
        assert np.array_equal(got, ref), (i, sh, zpA, zpW)


def test_eq2_equals_eq3(orc):
    """Eq. 2 (subtract first) == Eq. 3 (four terms) exactly, over every zp pair
    in the grid x random tiny shapes (reading R9)."""
    g = np.random.default_rng(21)
    for adt, wdt in [("u8", "s8"), ("u8", "u8"), ("s8", "s8")]:
        for zpA in ZPS[adt]:
            for zpW in ZPS[wdt]:
                for _ in range(8):
                    sh = _rand_shape(g)
                    A = gen.rand_q(g, (sh["N"], sh["C"], sh["H"], sh["W"]), adt)
                    W = gen.rand_q(g, (sh["K"], sh["C"] // sh["groups"], sh["R"], sh["S"]), wdt)
                    kw = dict(stride=sh["stride"], pad=sh["pad"], dil=sh["dil"], groups=sh["groups"])
                    assert np.array_equal(orc.conv2d_acc(A, W, zpA, zpW, **kw), orc.conv2d_eq3(A, W, zpA, zpW, **kw))


def test_explicit_zp_prepadding_equals_padding(orc):
    g = np.random.default_rng(22)
    A = gen.rand_q(g, (2, 3, 6, 7), "u8")
    W = gen.rand_q(g, (4, 3, 3, 3), "s8")
    zpA = 77
    Ap = np.full((2, 3, 6 + 3, 7 + 2), zpA, np.uint8)
    Ap[:, :, 1:7, 2:9] = A
    a = orc.conv2d_acc(A, W, zpA, 3, pad=(1, 2, 2, 0), stride=(2, 1))
    b = orc.conv2d_acc(Ap, W, zpA, 3, pad=(0, 0, 0, 0), stride=(2, 1))
    assert np.array_equal(a, b)


def test_zero_point_shift_invariance(orc):
    """(Q_A + d, zp_A + d) describes the same real tensor (Eq. 1) -> same acc."""
    g = np.random.default_rng(23)
    A = gen.rand_q(g, (1, 4, 5, 5), "u8", 0, 200)
    W = gen.rand_q(g, (3, 4, 3, 3), "u8", 0, 200)
    base = orc.conv2d_acc(A, W, 100, 90, pad=(1, 1, 1, 1))
    for d in (1, 17, 55):
        assert np.array_equal(base, orc.conv2d_acc((A + d).astype(np.uint8), W, 100 + d, 90, pad=(1, 1, 1, 1)))
        assert np.array_equal(base, orc.conv2d_acc(A, (W + d).astype(np.uint8), 100, 90 + d, pad=(1, 1, 1, 1)))


def test_depthwise_equals_single_channel_convs(orc):
    g = np.random.default_rng(24)
    C = 5
    A = gen.rand_q(g, (2, C, 7, 6), "u8")
    W = gen.rand_q(g, (C, 1, 3, 3), "s8")
    dw = orc.conv2d_acc(A, W, 9, 0, pad=(1, 1, 1, 1), stride=(2, 2), groups=C)
    for c in range(C):
        one = orc.conv2d_acc(np.ascontiguousarray(A[:, c:c + 1]), np.ascontiguousarray(W[c:c + 1]), 9, 0,
                             pad=(1, 1, 1, 1), stride=(2, 2))
        assert np.array_equal(dw[:, c:c + 1], one)


def test_dense_equals_1x1_conv_and_numpy(orc):
    g = np.random.default_rng(25)
    A = gen.rand_q(g, (9, 33), "u8")
    W = gen.rand_q(g, (7, 33), "s8")
    bias = g.integers(-99, 99, size=7).astype(np.int32)
    d = orc.dense_acc(A, W, 131, -3, bias)
    c = orc.conv2d_acc(A.reshape(9, 33, 1, 1), W.reshape(7, 33, 1, 1), 131, -3, bias)
    assert np.array_equal(d, c.reshape(9, 7))
    ref = (A.astype(np.int64) - 131) @ (W.astype(np.int64) + 3).T + bias
    assert np.array_equal(d, ref)


def test_sampled_equals_full(orc):
    g = np.random.default_rng(26)
    A = gen.rand_q(g, (2, 6, 9, 8), "u8")
    W = gen.rand_q(g, (4, 6, 3, 3), "s8")
    kw = dict(stride=(2, 1), pad=(1, 1, 1, 1))
    full = orc.conv2d_acc(A, W, 12, 2, None, **kw)
    idx = g.choice(full.size, 50, replace=False)
    assert np.array_equal(orc.conv2d_acc_at(A, W, 12, 2, idx, None, **kw), full.reshape(-1)[idx])
    Ad = gen.rand_q(g, (20, 31), "u8")
    Wd = gen.rand_q(g, (9, 31), "u8")
    fd = orc.dense_acc(Ad, Wd, 5, 200)
    idx = g.choice(fd.size, 40, replace=False)
    assert np.array_equal(orc.dense_acc_at(Ad, Wd, 5, 200, idx), fd.reshape(-1)[idx])


def test_requantized_conv_bounds_and_relu_commutation(orc):
    """Saturation: outputs in [qmin, qmax], >= zp_out with ReLU (invariant iii);
    ReLU before requantize == max(requantize, zp_out) (reading R6)."""
    for mode in ("upward", "tonearest"):
        c = gen.conv_case(31, 2, 16, 8, 8, 16, 3, 3, pad=(1, 1, 1, 1), relu=True, zp_out=20, rounding=mode)
        o = c.out_params()
        y = orc.qnn_conv2d(c.nchw(), c.oihw(), c.zp_A, c.zp_W, c.s_A, c.s_W, c.bias, o, pad=c.pad)
        assert y.min() >= 20 and y.max() <= 255
        o2 = dict(o, relu=False)
        y2 = orc.qnn_conv2d(c.nchw(), c.oihw(), c.zp_A, c.zp_W, c.s_A, c.s_W, c.bias, o2, pad=c.pad)
        assert np.array_equal(y, np.maximum(y2, 20))


def test_relu_commutes_on_random_accumulators(orc):
    """rq(max(v,0)) == max(rq(v), zp_out) on 10^5 random draws per mode (reading R6)."""
    g = np.random.default_rng(32)
    v = g.integers(-2 ** 31, 2 ** 31, size=100_000, dtype=np.int64)
    M = np.array([int(g.integers(2 ** 30, 2 ** 31))], np.int32)
    S = np.array([-7], np.int32)
    for mode in ("upward", "tonearest"):
        a = orc.requantize_acc(v, M, S, "s8", 5, mode, relu=True, axis=0)
        b = orc.requantize_acc(v, M, S, "s8", 5, mode, relu=False, axis=0)
        assert np.array_equal(a, np.maximum(b, 5))


def test_determinism(orc):
    c = gen.conv_case(33, 1, 8, 6, 6, 8, 3, 3, pad=(1, 1, 1, 1))
    a = orc.qnn_conv2d(c.nchw(), c.oihw(), c.zp_A, c.zp_W, c.s_A, c.s_W, c.bias, c.out_params(), pad=c.pad)
    b = orc.qnn_conv2d(c.nchw(), c.oihw(), c.zp_A, c.zp_W, c.s_A, c.s_W, c.bias, c.out_params(), pad=c.pad)
    assert a.tobytes() == b.tobytes()
