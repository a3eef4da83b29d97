"""GPU parity: qnn.add and pooling vs the oracle, bit-exact."""
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


@pytest.mark.parametrize("adt,bdt,odt", [("u8", "u8", "u8"), ("u8", "s8", "s8"), ("s8", "s8", "u8")])
@pytest.mark.parametrize("mode", ["upward", "tonearest"])
@pytest.mark.parametrize("relu", [False, True])
def test_add(q, adt, bdt, odt, mode, relu):
    g = np.random.default_rng(zlib.crc32(f"{adt}{bdt}{odt}{mode}{relu}".encode()))
    for n in (1, 15, 16, 4097, 256 * 56 * 56):
        a = gen.rand_q(g, (n,), adt)
        b = gen.rand_q(g, (n,), bdt)
        s_a, s_b, s_o = (float(np.float32(v)) for v in g.uniform(0.01, 0.3, 3))
        za = int(g.integers(0, 256)) if adt == "u8" else int(g.integers(-128, 128))
        zb = int(g.integers(0, 256)) if bdt == "u8" else int(g.integers(-128, 128))
        zo = int(g.integers(0, 256)) if odt == "u8" else int(g.integers(-128, 128))
        want = orc.add(a, s_a, za, b, s_b, zb, s_o, zo, odt, mode, relu)
        got = q.qnn_add(torch.from_numpy(a).cuda(), s_a, za, torch.from_numpy(b).cuda(), s_b, zb, s_o, zo, odt,
                        mode, relu).cpu().numpy()
        assert np.array_equal(got, want), (n, np.argwhere(got != want)[:5])


def test_add_unaligned(q):
    g = np.random.default_rng(5)
    base_a = torch.from_numpy(gen.rand_q(g, (5000,), "u8")).cuda()
    base_b = torch.from_numpy(gen.rand_q(g, (5000,), "u8")).cuda()
    a, b = base_a[3:3 + 4001], base_b[7:7 + 4001]
    want = orc.add(a.cpu().numpy(), 0.05, 3, b.cpu().numpy(), 0.07, 200, 0.1, 128, "u8")
    got = q.qnn_add(a, 0.05, 3, b, 0.07, 200, 0.1, 128, "u8").cpu().numpy()
    assert np.array_equal(got, want)


POOLS = [
    # N, H, W, C, R, S, stride, pad, mode, dtype
    (2, 112, 112, 64, 3, 3, (2, 2), (1, 1, 1, 1), "max", "u8"),     # ResNet-50 stem max pool
    (4, 7, 7, 2048, 7, 7, (1, 1), (0, 0, 0, 0), "avg", "u8"),       # ResNet-50 global average pool
    (2, 8, 8, 2048, 8, 8, (1, 1), (0, 0, 0, 0), "avg", "s8"),       # Inception-v3 global pool
    (2, 35, 35, 48, 3, 3, (1, 1), (1, 1, 1, 1), "avg", "u8"),       # Inception branch pool, padded
    (1, 13, 11, 5, 3, 2, (2, 1), (1, 0, 1, 1), "max", "s8"),        # odd shapes: scalar path
    (1, 9, 9, 7, 2, 2, (2, 2), (0, 0, 1, 1), "avg", "s8"),
]


POOLS += [
    # the fast 16-channel kernel at network shapes (ragged Q vs its 4-column blocks), both dtypes
    (2, 35, 35, 256, 3, 3, (1, 1), (1, 1, 1, 1), "avg", "u8"),     # Inception branch avg pool
    (2, 35, 35, 48, 3, 3, (1, 1), (1, 1, 1, 1), "avg", "s8"),
    (2, 147, 147, 64, 3, 3, (2, 2), (0, 0, 0, 0), "max", "u8"),    # Inception stem max pool
    (2, 112, 112, 64, 3, 3, (2, 2), (1, 1, 1, 1), "max", "s8"),    # ResNet-50 stem max pool
    (3, 8, 8, 2048, 8, 8, (1, 1), (0, 0, 0, 0), "avg", "u8"),      # Inception global avg pool
    (3, 7, 7, 2048, 7, 7, (1, 1), (0, 0, 0, 0), "avg", "s8"),      # ResNet-50 global avg pool
    (1, 17, 13, 32, 5, 3, (2, 1), (2, 1, 1, 0), "avg", "u8"),      # asymmetric everything
    (1, 9, 11, 16, 11, 11, (1, 1), (5, 5, 5, 5), "avg", "s8"),     # 121 taps: the 16-bit lane limit side
]


@pytest.mark.parametrize("cfg", POOLS, ids=lambda c: f"{c[8]}_{c[1]}x{c[2]}x{c[3]}_k{c[4]}{c[5]}")
def test_pool(q, cfg):
    N, H, W, C, R, S, st, pad, mode, dt = cfg
    g = np.random.default_rng(zlib.crc32(str(cfg).encode()))
    x = gen.rand_q(g, (N, H, W, C), dt)
    want = orc.pool2d(np.ascontiguousarray(x.transpose(0, 3, 1, 2)), mode, R, S, st, pad).transpose(0, 2, 3, 1)
    got = q.qnn_pool2d(torch.from_numpy(x).cuda(), mode, R, S, st, pad).cpu().numpy()
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- conv + fused residual add
FUSED = [
    # N, C, H, W, K, R, stride, pad, res_dtype, out_dtype, relu, mode
    (2, 64, 14, 14, 256, 1, (1, 1), (0, 0, 0, 0), "u8", "u8", True, "upward"),      # bottleneck conv3
    (3, 32, 11, 13, 64, 3, (1, 1), (1, 1, 1, 1), "u8", "u8", True, "upward"),       # border classes
    (2, 48, 9, 9, 96, 3, (2, 2), (1, 1, 1, 1), "s8", "s8", False, "tonearest"),
    (1, 128, 7, 7, 512, 1, (1, 1), (0, 0, 0, 0), "u8", "u8", False, "upward"),      # 2 N tiles
    (2, 16, 10, 10, 32, 3, (1, 1), (1, 1, 1, 1), "u8", "u8", True, "tonearest"),
    # channel-major pointwise kernel with the residual tile staged by TMA
    (3, 256, 9, 11, 1024, 1, (1, 1), (0, 0, 0, 0), "s8", "u8", True, "upward"),
    (2, 128, 10, 10, 256, 1, (1, 1), (0, 0, 0, 0), "u8", "s8", False, "tonearest"),
    (1, 1024, 5, 5, 256, 1, (1, 1), (0, 0, 0, 0), "u8", "u8", True, "upward"),      # streamed weights
]


@pytest.mark.parametrize("cfg", FUSED, ids=lambda c: f"C{c[1]}K{c[4]}_{c[2]}x{c[3]}_r{c[5]}_{c[8]}{c[9]}_{c[11]}")
def test_conv_fused_residual_add(q, cfg):
    from gpu_helpers import to_dev
    N, C, H, W, K, R, st, pad, rdt, odt, relu, mode = cfg
    case = gen.conv_case(1300 + C + K, N, C, H, W, K, R, R, st, pad, (1, 1), 1, "u8", "s8", out_dtype=odt,
                         relu=relu, rounding=mode, zp_out=5 if odt == "u8" else -3)
    P, Q = orc.out_hw(H, W, R, R, st, pad)
    g = np.random.default_rng(zlib.crc32(str(cfg).encode()))
    res = gen.rand_q(g, (N, P, Q, K), rdt)
    s_res, zp_res = 0.7 * case.s_out, (117 if rdt == "u8" else -9)
    op = q.PackedConv2d(N, H, W, C, to_dev(case.W), to_dev(case.bias), case.zp_A, case.zp_W, case.s_A, case.s_W,
                        case.out_params(), case.stride, case.pad, (1, 1), 1)
    y = op(to_dev(case.A), residual=(to_dev(res), s_res, zp_res)).cpu().numpy()
    want = orc.qnn_conv2d_add(case.nchw(), case.oihw(), case.zp_A, case.zp_W, case.s_A, case.s_W, case.bias,
                              np.ascontiguousarray(res.transpose(0, 3, 1, 2)), s_res, zp_res, case.out_params(),
                              case.stride, case.pad).transpose(0, 2, 3, 1)
    assert np.array_equal(y, want), (np.argwhere(y != want)[:5], y.size)


def test_pool_into_channel_slice(q):
    """Pooling written into channels [96, 96 + C) of a wider concat buffer (Inception reduction
    blocks); the other channels stay untouched."""
    g = np.random.default_rng(77)
    x = gen.rand_q(g, (2, 17, 17, 64), "u8")
    want = orc.pool2d(np.ascontiguousarray(x.transpose(0, 3, 1, 2)), "max", 3, 3, (2, 2)).transpose(0, 2, 3, 1)
    buf = torch.full((2, 8, 8, 256), 7, dtype=torch.uint8, device="cuda")
    q.qnn_pool2d(torch.from_numpy(x).cuda(), "max", 3, 3, (2, 2), out=buf, out_channel_offset=96)
    b = buf.cpu().numpy()
    assert np.array_equal(b[..., 96:160], want)
    assert (b[..., :96] == 7).all() and (b[..., 160:] == 7).all()
