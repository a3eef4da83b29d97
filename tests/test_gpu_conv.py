"""GPU parity: qnn.conv2d (tcgen05 implicit GEMM + fused epilogue) and the
depthwise kernel vs the oracle, bit-exact, on seeded inputs.

Coverage: BASELINE config 1 (both outputs, both rounding modes, pad 0/1);
random shapes spanning several 128-row tiles with ragged tails, strides,
dilation, asymmetric padding, u8/s8 operands, zp_W != 0 (Term 3 row sums),
channel counts that need the padded-pitch copy, K not a multiple of 32,
multiple N tiles, raw int32 output, a channel-strided output; ResNet-50 and
MobileNet-v2 layer shapes (full compare at batch 1, sampled at batch 64/128).
"""
import zlib

import numpy as np
import pytest
import torch

import oracle as orc
from gpu_helpers import gpu_conv, mismatch_report, oracle_conv, oracle_conv_at
from workloads import gen
from workloads.shapes import inception_v3_convs, mobilenet_v2_convs, resnet50_unique

pytestmark = pytest.mark.gpu


def config1_case(pad, relu, mode):
    """BASELINE.json configs[0]: N=1, C=16, H=W=8, K=16, 3x3, u8 input zp=128,
    s8 per-channel weights, requantize to u8 (reading R18 for the unstated details)."""
    g = np.random.default_rng(101)
    A = gen.rand_q(g, (1, 8, 8, 16), "u8")
    W = gen.rand_q(np.random.default_rng(102), (16, 3, 3, 16), "s8", -127, 127)
    k = np.arange(16)
    s_W = np.where(k < 8, 2.0 ** -7 * 2.0 ** -(k % 4), 0.0037 * (1 + k / 16)).astype(np.float32)
    bias = np.random.default_rng(103).integers(-4096, 4097, size=16).astype(np.int32)
    return gen.ConvCase(A, W, bias, 128, 0, 0.5, s_W, 4.0, 0 if relu else 128, "u8", (1, 1), (pad,) * 4, (1, 1), 1,
                        relu, None, None, mode)


@pytest.mark.parametrize("pad", [1, 0])
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("mode", ["upward", "tonearest"])
def test_config1(pad, relu, mode):
    case = config1_case(pad, relu, mode)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert got.shape == want.shape
    assert np.array_equal(got, want), mismatch_report(got, want)


SWEEP = [
    # N, C, H, W, K, R, S, stride, pad(t,l,b,r), dil, a, w, zpW, out, per_channel
    (2, 16, 9, 11, 16, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), "u8", "s8", 0, "u8", True),
    (3, 64, 20, 19, 64, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), "u8", "s8", 0, "u8", True),
    (2, 64, 17, 17, 96, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), "u8", "s8", 0, "s8", True),
    (2, 128, 15, 15, 256, 1, 1, (2, 2), (0, 0, 0, 0), (1, 1), "u8", "s8", 0, "u8", True),
    (1, 32, 23, 21, 48, 5, 5, (1, 1), (2, 2, 2, 2), (1, 1), "u8", "s8", 0, "u8", True),
    (2, 48, 13, 14, 64, 3, 3, (2, 2), (1, 1, 1, 1), (1, 1), "s8", "s8", 0, "s8", True),
    (2, 32, 12, 12, 40, 3, 3, (1, 1), (2, 2, 2, 2), (2, 2), "u8", "s8", 0, "u8", True),
    (1, 80, 10, 17, 100, 1, 7, (1, 1), (0, 3, 0, 3), (1, 1), "u8", "s8", 0, "u8", True),
    (1, 80, 17, 10, 100, 7, 1, (1, 1), (3, 0, 3, 0), (1, 1), "u8", "s8", 0, "u8", True),
    (2, 64, 11, 9, 64, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), "u8", "u8", 117, "u8", False),   # TFLite u8 x u8
    (2, 96, 14, 14, 300, 3, 3, (2, 2), (0, 1, 1, 0), (1, 1), "u8", "u8", 131, "u8", False),  # asym pad, 2 N tiles
    (1, 3, 30, 30, 32, 7, 7, (2, 2), (3, 3, 3, 3), (1, 1), "u8", "s8", 0, "u8", True),     # stem: pad-copy
    (2, 24, 16, 16, 72, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), "u8", "s8", 0, "u8", True),    # C=24: pad-copy, 2-D A
    (1, 144, 9, 9, 24, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), "s8", "s8", -7, "s8", True),
    (2, 256, 7, 7, 512, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), "u8", "s8", 0, "u8", True),
    (1, 64, 8, 8, 1000, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), "u8", "s8", 0, "u8", True),    # K=1000 tail
    (2, 32, 10, 10, 64, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), "u8", "s8", 0, "s32", True),   # raw int32
    (1, 16, 5, 5, 16, 5, 5, (1, 1), (0, 0, 0, 0), (1, 1), "u8", "s8", 3, "s32", True),     # 1x1 output, raw
    # Term-3 pixel sums on the coalesced path (C / 16 a power of two: 1, 16, 128 chunks per pixel)
    (2, 256, 7, 9, 64, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), "s8", "u8", 77, "u8", False),
    (1, 2048, 5, 5, 32, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), "s8", "s8", -5, "s8", True),
    (3, 16, 6, 7, 16, 3, 3, (2, 2), (1, 1, 1, 1), (1, 1), "u8", "s8", 9, "u8", True),
    # ... and with C / 16 not a power of two (Inception-v3 widths: 12 and 48 chunks per pixel)
    (1, 192, 9, 11, 64, 1, 7, (1, 1), (0, 3, 0, 3), (1, 1), "u8", "u8", 100, "u8", False),
    (2, 768, 5, 5, 32, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), "s8", "s8", 4, "s8", True),
]


@pytest.mark.parametrize("i", range(len(SWEEP)))
def test_conv_sweep(i):
    N, C, H, W, K, R, S, st, pad, dil, adt, wdt, zpW, odt, pc = SWEEP[i]
    for mode in ("upward", "tonearest"):
        case = gen.conv_case(500 + i, N, C, H, W, K, R, S, st, pad, dil, 1, adt, wdt, zp_W=zpW, per_channel=pc,
                             out_dtype=odt, relu=(i % 2 == 0), rounding=mode)
        _, _, y = gpu_conv(case)
        got, want = y.cpu().numpy(), oracle_conv(case)
        assert np.array_equal(got, want), f"{SWEEP[i]} {mode}\n" + mismatch_report(got, want)


@pytest.mark.parametrize("mode", ["upward", "tonearest"])
def test_conv_generic_requant_path(mode):
    """Channels whose multiplier is outside the epilogue's mulhi fast range
    (m >= 2^-1, i.e. right shift <= 32, or m < 2^-21) force the generic 64-bit
    rounding for the whole tile; small operands keep outputs unsaturated."""
    g = np.random.default_rng(91)
    N, H, W, C, K = 2, 9, 9, 32, 64
    A = (128 + g.integers(-3, 4, size=(N, H, W, C))).astype(np.uint8)
    Wt = g.integers(-1, 2, size=(K, 3, 3, C)).astype(np.int8)
    s_A, s_out = 0.05, 0.04
    s_W = np.full(K, 0.003, np.float32)
    s_W[0] = 0.9            # m = 1.125 -> shift 1  (rsh 30)
    s_W[1] = 0.5            # m = 0.625 -> rsh 31
    s_W[2] = 0.33           # m ~ 0.41  -> rsh 32
    s_W[3] = 1e-7           # m ~ 1.2e-7 -> rsh 54 (> 52)
    bias = g.integers(-20, 21, size=K).astype(np.int32)
    case = gen.ConvCase(A, Wt, bias, 128, 0, s_A, s_W, s_out, 128, "u8", (1, 1), (1, 1, 1, 1), (1, 1), 1, False,
                        None, None, mode)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), mismatch_report(got, want)
    assert len(np.unique(want[..., 0])) > 5          # channel 0 is not saturated


def test_conv_strided_output_and_determinism():
    case = gen.conv_case(77, 2, 32, 12, 12, 48, 3, 3, (1, 1), (1, 1, 1, 1))
    _, x, y = gpu_conv(case, out_cstride=80)
    got = y.cpu().numpy()[..., :48]
    assert np.array_equal(got, oracle_conv(case))
    op, x, y2 = gpu_conv(case, out_cstride=80)
    y3 = op(x)
    torch.cuda.synchronize()
    assert np.array_equal(y2.cpu().numpy()[..., :48], y3.cpu().numpy()[..., :48])


def test_conv_batch_shard_invariance():
    """Images are independent: conv of a batch == concat of per-shard convs."""
    case = gen.conv_case(78, 4, 64, 14, 14, 64, 3, 3, (1, 1), (1, 1, 1, 1))
    _, _, y = gpu_conv(case)
    full = y.cpu().numpy()
    for lo, hi in [(0, 1), (1, 3), (3, 4)]:
        sub = gen.ConvCase(**{**case.__dict__, "A": case.A[lo:hi]})
        _, _, ys = gpu_conv(sub)
        assert np.array_equal(ys.cpu().numpy(), full[lo:hi])


@pytest.mark.parametrize("layer", resnet50_unique(), ids=lambda c: c.name)
def test_resnet50_layers_batch1_full(layer):
    case = gen.conv_case(1000 + zlib.crc32(layer.name.encode()) % 1000, 1, layer.C, layer.H, layer.W, layer.K, layer.R, layer.S,
                         layer.stride, layer.pad, (1, 1), 1, "u8", "s8", relu=layer.relu)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), layer.name + "\n" + mismatch_report(got, want)


@pytest.mark.parametrize("layer", [c for c in resnet50_unique() if c.name in
                                   ("conv1", "layer1.0.conv2", "layer2.0.conv2", "layer3.1.conv1", "layer4.0.downsample",
                                    "layer4.1.conv2")], ids=lambda c: c.name)
@pytest.mark.parametrize("per_channel", [True, False])
def test_resnet50_layers_batch64_sampled(layer, per_channel):
    """Full-size (batch 64) launch; 4096 sampled outputs checked against the oracle
    (per-tensor variant uses TFLite-style u8 weights with zp_W != 0)."""
    wdt, zpW = ("s8", 0) if per_channel else ("u8", 128 + (zlib.crc32(layer.name.encode()) % 29) - 14)
    case = gen.conv_case(2000 + zlib.crc32(layer.name.encode()) % 1000, 64, layer.C, layer.H, layer.W, layer.K, layer.R, layer.S,
                         layer.stride, layer.pad, (1, 1), 1, "u8", wdt, zp_W=zpW, per_channel=per_channel,
                         relu=layer.relu)
    _, _, y = gpu_conv(case)
    got = y.cpu().numpy().reshape(-1)
    g = np.random.default_rng(3)
    idx = g.choice(got.size, 4096, replace=False)
    idx[:8] = [0, 1, got.size - 1, got.size - 2, layer.K - 1, layer.K, got.size // 2, got.size - layer.K]
    want = oracle_conv_at(case, idx, layer.P, layer.Q)
    assert np.array_equal(got[idx], want), layer.name


def _inception_unique():
    out, seen = [], set()
    for c in inception_v3_convs():
        k = (c.C, c.K, c.H, c.W, c.R, c.S, c.stride, c.pad)
        if k not in seen:
            seen.add(k)
            out.append(c)
    return out


@pytest.mark.parametrize("layer", _inception_unique(), ids=lambda c: c.name)
def test_inception_v3_layers_batch1_full(layer):
    """BASELINE configs[4]'s Inception-v3 stack: every distinct conv shape (3x3/s2/p0 stems,
    5x5/p2 with 25 border classes, 1x7 / 7x1 and 1x3 / 3x1 asymmetric padding), full compare."""
    case = gen.conv_case(3000 + zlib.crc32(layer.name.encode()) % 1000, 1, layer.C, layer.H, layer.W, layer.K,
                         layer.R, layer.S, layer.stride, layer.pad, (1, 1), 1, "u8", "s8", relu=layer.relu)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), layer.name + "\n" + mismatch_report(got, want)


@pytest.mark.parametrize("layer", [c for c in _inception_unique() if c.name in
                                   ("Conv2d_2b_3x3", "Mixed_5b.branch5x5_2", "Mixed_6b.branch7x7_2",
                                    "Mixed_6b.branch7x7_3", "Mixed_7b.branch3x3_2a", "Mixed_7c.branch1x1")],
                         ids=lambda c: c.name)
def test_inception_v3_layers_batch64_sampled(layer):
    """Full-size (batch 64) Inception-v3 launches, 4096 sampled outputs vs the oracle."""
    case = gen.conv_case(4000 + zlib.crc32(layer.name.encode()) % 1000, 64, layer.C, layer.H, layer.W, layer.K,
                         layer.R, layer.S, layer.stride, layer.pad, (1, 1), 1, "u8", "s8", relu=layer.relu)
    _, _, y = gpu_conv(case)
    got = y.cpu().numpy().reshape(-1)
    idx = np.random.default_rng(5).choice(got.size, 4096, replace=False)
    idx[:6] = [0, 1, got.size - 1, layer.K - 1, layer.K, got.size - layer.K]
    want = oracle_conv_at(case, idx, layer.P, layer.Q)
    assert np.array_equal(got[idx], want), layer.name


def _mobilenet_dense_unique():
    out, seen = [], set()
    for c in mobilenet_v2_convs():
        k = (c.C, c.K, c.H, c.W, c.R, c.S, c.stride, c.act6, c.relu)
        if c.groups == 1 and k not in seen:
            seen.add(k)
            out.append(c)
    return out


@pytest.mark.parametrize("layer", _mobilenet_dense_unique(), ids=lambda c: c.name)
def test_mobilenet_v2_pointwise_batch2_full(layer):
    """BASELINE configs[2]'s non-depthwise MobileNet-v2 convs (3x3/s2 stem, 1x1 expand with
    ReLU6 as an output-domain clamp, 1x1 linear project, last 1x1), full compare at batch 2."""
    case = gen.conv_case(5000 + zlib.crc32(layer.name.encode()) % 1000, 2, layer.C, layer.H, layer.W, layer.K,
                         layer.R, layer.S, layer.stride, layer.pad, (1, 1), 1, "u8", "s8", relu=layer.relu,
                         act6=layer.act6)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), layer.name + "\n" + mismatch_report(got, want)


def _dw_layers():
    out, seen = [], set()
    for c in mobilenet_v2_convs():
        if c.groups > 1 and (c.C, c.stride) not in seen:
            seen.add((c.C, c.stride))
            out.append(c)
    return out


@pytest.mark.parametrize("C,stride,act6,adt", [(16, 1, True, "u8"), (32, 2, False, "u8"), (144, 1, True, "u8"),
                                               (12, 1, False, "s8"), (7, 2, True, "u8"), (96, 2, True, "s8")])
def test_depthwise_small(C, stride, act6, adt):
    for mode in ("upward", "tonearest"):
        case = gen.conv_case(600 + C, 2, C, 13, 15, C, 3, 3, (stride, stride), (1, 1, 1, 1), (1, 1), C, adt, "s8",
                             relu=True, act6=act6, rounding=mode)
        _, _, y = gpu_conv(case)
        got, want = y.cpu().numpy(), oracle_conv(case)
        assert np.array_equal(got, want), mismatch_report(got, want)


def test_depthwise_zpW_and_raw():
    case = gen.conv_case(650, 1, 32, 9, 9, 32, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), 32, "u8", "u8", zp_W=120,
                         per_channel=False, out_dtype="s32")
    _, _, y = gpu_conv(case)
    assert np.array_equal(y.cpu().numpy(), oracle_conv(case))


@pytest.mark.parametrize("layer", _dw_layers(), ids=lambda c: f"{c.name}_C{c.C}_s{c.stride[0]}")
def test_mobilenet_depthwise_batch128_sampled(layer):
    case = gen.conv_case(3000 + layer.C, 128, layer.C, layer.H, layer.W, layer.K, 3, 3, layer.stride, layer.pad,
                         (1, 1), layer.C, "u8", "s8", relu=True, act6=True)
    _, _, y = gpu_conv(case)
    got = y.cpu().numpy().reshape(-1)
    idx = np.random.default_rng(4).choice(got.size, 4096, replace=False)
    want = oracle_conv_at(case, idx, layer.P, layer.Q)
    assert np.array_equal(got[idx], want)


def test_errors_raise():
    from paper_2006_10226_b200 import QnnError
    case = gen.conv_case(700, 1, 8, 6, 6, 8, 3, 3, (1, 1), (1, 1, 1, 1), groups=2)
    with pytest.raises(QnnError):
        gpu_conv(case)


# tensor-core depthwise path (C % 32 == 0, s8 weights, zp_W == 0, stride 1/2, 8-bit output):
# several strips and 128-row tiles, wide rows (Wp > 128), 5x5, asymmetric padding, clamps
DW_TC = [
    # N, C, H, W, R, stride, pad(t,l,b,r), a_dtype, out_dtype, act6, mode
    (2, 32, 30, 37, 3, 1, (1, 1, 1, 1), "u8", "u8", True, "upward"),
    (1, 64, 7, 7, 3, 1, (1, 1, 1, 1), "u8", "u8", True, "upward"),
    (3, 96, 14, 14, 3, 2, (1, 1, 1, 1), "u8", "u8", True, "upward"),
    (1, 32, 57, 150, 3, 1, (1, 1, 1, 1), "u8", "u8", False, "upward"),
    (2, 64, 19, 23, 5, 1, (2, 2, 2, 2), "s8", "s8", False, "upward"),
    (2, 32, 20, 21, 5, 2, (2, 2, 2, 2), "u8", "u8", True, "tonearest"),
    (1, 160, 15, 16, 3, 2, (0, 0, 1, 1), "u8", "s8", False, "tonearest"),
    (4, 32, 9, 9, 3, 1, (0, 0, 0, 0), "u8", "u8", True, "upward"),
]


@pytest.mark.parametrize("cfg", DW_TC, ids=lambda c: f"C{c[1]}_{c[2]}x{c[3]}_r{c[4]}_s{c[5]}_{c[10]}")
def test_depthwise_tensor_core_path(cfg):
    N, C, H, W, R, st, pad, adt, odt, act6, mode = cfg
    case = gen.conv_case(800 + C + H, N, C, H, W, C, R, R, (st, st), pad, (1, 1), C, adt, "s8", out_dtype=odt,
                         relu=True, act6=act6, rounding=mode, zp_out=0 if odt == "u8" else -5)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), mismatch_report(got, want)


def test_depthwise_forced_kernels_subprocess():
    """The 3x3 shapes normally take the TMA-staged kernel; run the register-blocked dp4a, the
    tensor-core and the generic kernels on them too (QNN_DW_IMPL is read once per process,
    hence the subprocess)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
from gpu_helpers import gpu_conv, oracle_conv
from workloads import gen
for cfg in [(2, 32, 30, 37, 1, "upward"), (3, 96, 14, 14, 2, "tonearest"), (1, 48, 11, 13, 1, "upward")]:
    N, C, H, W, st, mode = cfg
    case = gen.conv_case(900 + C, N, C, H, W, C, 3, 3, (st, st), (1, 1, 1, 1), (1, 1), C, "u8", "s8",
                         relu=True, act6=True, rounding=mode)
    _, _, y = gpu_conv(case)
    assert np.array_equal(y.cpu().numpy(), oracle_conv(case)), cfg
print("OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for impl in ("dp4a", "tc", "generic"):
        env = dict(os.environ, QNN_DW_IMPL=impl)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0 and "OK" in r.stdout, (impl, r.stdout[-2000:], r.stderr[-2000:])


# width-folded small-C convolutions (stems): the GEMM builds X' tiles in shared memory
FOLD_CASES = [
    # N, C, H, W, K, R, S, stride, pad(t,l,b,r), dil, a_dtype, w_dtype, zp_W
    (2, 3, 33, 35, 64, 7, 7, (2, 2), (3, 3, 3, 3), (1, 1), "u8", "s8", 0),
    (1, 4, 17, 19, 32, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), "s8", "s8", 0),
    (2, 8, 15, 13, 48, 3, 3, (2, 2), (1, 0, 1, 2), (1, 1), "u8", "s8", 0),
    (1, 3, 20, 21, 16, 5, 5, (1, 1), (2, 2, 2, 2), (1, 2), "u8", "s8", 0),
    (1, 6, 12, 12, 40, 5, 5, (1, 1), (2, 2, 2, 2), (1, 1), "u8", "s8", 0),
    (3, 3, 9, 9, 64, 7, 7, (2, 2), (3, 3, 3, 3), (1, 1), "u8", "s8", 0),
    (2, 3, 23, 24, 32, 3, 3, (2, 2), (1, 1, 1, 1), (1, 1), "u8", "u8", 119),
    # W*C % 16 == 0: X' tiles built in shared memory from TMA-staged raw rows
    (2, 3, 37, 32, 64, 7, 7, (2, 2), (3, 3, 3, 3), (1, 1), "u8", "s8", 0),
    (1, 4, 20, 24, 32, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), "s8", "s8", 0),
    (2, 8, 15, 14, 48, 3, 3, (2, 2), (1, 0, 1, 2), (1, 1), "u8", "s8", 0),
    (1, 6, 16, 16, 40, 5, 5, (1, 1), (2, 2, 2, 2), (1, 1), "u8", "s8", 0),
    (3, 3, 16, 16, 64, 7, 7, (2, 2), (3, 3, 3, 3), (1, 1), "u8", "s8", 0),
    (2, 3, 32, 32, 32, 3, 3, (2, 2), (1, 1, 1, 1), (1, 1), "u8", "u8", 119),
    (1, 4, 20, 20, 16, 3, 3, (1, 1), (2, 1, 2, 1), (2, 1), "u8", "s8", 0),
    (1, 3, 64, 224, 64, 7, 7, (2, 2), (3, 3, 3, 3), (1, 1), "u8", "s8", 0),
]


@pytest.mark.parametrize("cfg", FOLD_CASES, ids=lambda c: f"C{c[1]}_{c[2]}x{c[3]}_k{c[5]}x{c[6]}_s{c[7][0]}")
def test_folded_small_channel_conv(cfg):
    N, C, H, W, K, R, S, st, pad, dil, adt, wdt, zpW = cfg
    case = gen.conv_case(1100 + C * 7 + H, N, C, H, W, K, R, S, st, pad, dil, 1, adt, wdt, zp_W=zpW,
                         per_channel=zpW == 0)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), mismatch_report(got, want)


def test_folded_conv_hbm_copy_path_subprocess():
    """QNN_NO_ABUILD=1 takes the materialised-X' path (fold kernel + TMA im2col) instead."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
from gpu_helpers import gpu_conv, oracle_conv
from workloads import gen
case = gen.conv_case(1200, 2, 3, 33, 35, 64, 7, 7, (2, 2), (3, 3, 3, 3), (1, 1), 1, "u8", "s8")
_, _, y = gpu_conv(case)
assert np.array_equal(y.cpu().numpy(), oracle_conv(case))
print("OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, QNN_NO_ABUILD="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


# TMA-staged 3x3 depthwise: channel slices (CS 16/32/64), multi-band images, odd widths, pad
# variants, zp_W != 0 (weights W - zp_W still in s8), s8 activations, last partial bands
DWT_CASES = [
    # N, C, H, W, stride, pad, a_dtype, w_dtype, zp_W, out, rounding
    (2, 32, 40, 37, 1, (1, 1, 1, 1), "u8", "s8", 0, "u8", "upward"),
    (2, 144, 19, 21, 1, (1, 1, 1, 1), "u8", "s8", 0, "u8", "upward"),     # CS 16
    (1, 192, 29, 23, 2, (1, 1, 1, 1), "u8", "s8", 0, "u8", "upward"),     # CS 64, stride 2, odd
    (3, 96, 17, 17, 2, (0, 0, 1, 1), "s8", "s8", 0, "s8", "upward"),      # asymmetric pad
    (2, 64, 13, 9, 1, (0, 0, 0, 0), "u8", "u8", 121, "u8", "upward"),     # no pad, zp_W
    (1, 48, 33, 30, 1, (1, 1, 1, 1), "u8", "s8", 0, "u8", "tonearest"),   # generic rounding path
    (1, 32, 112, 112, 1, (1, 1, 1, 1), "u8", "s8", 0, "u8", "upward"),    # MobileNet block0 shape
]


@pytest.mark.parametrize("cfg", DWT_CASES, ids=lambda c: f"C{c[1]}_{c[2]}x{c[3]}_s{c[4]}_{c[10]}")
def test_depthwise_tma_staged(cfg):
    N, C, H, W, st, pad, adt, wdt, zpW, odt, mode = cfg
    case = gen.conv_case(1500 + C + H, N, C, H, W, C, 3, 3, (st, st), pad, (1, 1), C, adt, wdt, zp_W=zpW,
                         per_channel=zpW == 0, out_dtype=odt, relu=True, act6=(C % 64 == 0), rounding=mode)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), mismatch_report(got, want)


# stride-1 convolutions with resident weights: per (tile, channel chunk) one TMA box of the
# input rows the tile touches; every tap is an MMA whose A descriptor starts (r*Wp + s) rows in
AROWS_CASES = [
    # N, C, H, W, K, R, S, pad(t,l,b,r), a_dtype, w_dtype, zp_W, out
    (2, 64, 20, 19, 64, 3, 3, (1, 1, 1, 1), "u8", "s8", 0, "u8"),      # BK 64 (SW64)
    (2, 128, 14, 15, 128, 3, 3, (1, 1, 1, 1), "u8", "s8", 0, "u8"),    # BK 128 (SW128)
    (3, 32, 9, 7, 48, 3, 3, (1, 1, 1, 1), "s8", "s8", 0, "s8"),        # BK 32, Wp 9 (many rows per tile)
    (1, 64, 56, 56, 64, 3, 3, (1, 1, 1, 1), "u8", "s8", 0, "u8"),      # ResNet layer1 conv2
    (2, 64, 11, 9, 64, 3, 3, (1, 1, 1, 1), "u8", "u8", 117, "u8"),     # zp_W != 0 (row sums)
    (1, 32, 23, 21, 48, 5, 5, (2, 2, 2, 2), "u8", "s8", 0, "u8"),      # 5x5
    (1, 64, 10, 17, 96, 1, 7, (0, 3, 0, 3), "u8", "s8", 0, "u8"),      # 1x7
    (1, 64, 17, 10, 96, 7, 1, (3, 0, 3, 0), "u8", "s8", 0, "s8"),      # 7x1
    (2, 64, 13, 12, 64, 3, 3, (0, 2, 1, 0), "u8", "s8", 0, "u8"),      # asymmetric pad
    (1, 64, 6, 200, 32, 3, 3, (1, 1, 1, 1), "u8", "s8", 0, "u8"),      # wide rows: Wp 202
    (2, 96, 8, 8, 64, 3, 3, (1, 1, 1, 1), "u8", "s8", 0, "s32"),       # raw int32, 3 chunks of 32
    (2, 256, 7, 7, 256, 3, 3, (1, 1, 1, 1), "u8", "s8", 0, "u8"),      # 2 chunks of 128
]


@pytest.mark.parametrize("cfg", AROWS_CASES, ids=lambda c: f"C{c[1]}_{c[2]}x{c[3]}_k{c[5]}x{c[6]}_{c[11]}")
@pytest.mark.parametrize("mode", ["upward", "tonearest"])
def test_stride1_staged_rows_conv(cfg, mode):
    N, C, H, W, K, R, S, pad, adt, wdt, zpW, odt = cfg
    case = gen.conv_case(1300 + C + H * 3 + W, N, C, H, W, K, R, S, (1, 1), pad, (1, 1), 1, adt, wdt, zp_W=zpW,
                         per_channel=zpW == 0, out_dtype=odt, relu=(C % 64 == 0), rounding=mode)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), mismatch_report(got, want)


def test_stride1_im2col_path_subprocess():
    """QNN_NO_AROWS=1 keeps the per-tap TMA im2col path for the same stride-1 shapes."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
from gpu_helpers import gpu_conv, oracle_conv
from workloads import gen
for i, (C, H, W) in enumerate([(64, 20, 19), (128, 9, 11)]):
    case = gen.conv_case(1400 + i, 2, C, H, W, 64, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), 1, "u8", "s8")
    _, _, y = gpu_conv(case)
    assert np.array_equal(y.cpu().numpy(), oracle_conv(case))
print("OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, QNN_NO_AROWS="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


# wide pointwise convs on the channel-major GEMM (gemm_t.cu): output channels on the TMEM
# lanes; ragged pixel tails, 1..4 k-blocks, every BK, s8 in/out, clamps, TONEAREST (generic)
TRANS_CASES = [
    # N, C, H, W, K, a_dtype, out, relu, act6, rounding
    (2, 64, 9, 9, 256, "u8", "u8", True, False, "upward"),
    (1, 128, 28, 28, 512, "u8", "u8", True, False, "upward"),
    (2, 256, 14, 14, 1024, "s8", "s8", False, False, "upward"),
    (1, 512, 7, 7, 2048, "u8", "u8", True, False, "upward"),
    (3, 96, 5, 7, 384, "u8", "u8", True, True, "upward"),       # BK 32 x 3 chunks, clamp
    (2, 64, 6, 11, 256, "u8", "u8", True, False, "tonearest"),  # per-lane generic rounding
    (1, 640, 4, 4, 256, "u8", "s8", False, False, "upward"),    # 5 k-blocks of 128
    (2, 256, 19, 21, 128, "u8", "u8", True, False, "upward"),   # one channel block (K 128)
    (2, 1024, 7, 9, 256, "u8", "u8", True, False, "upward"),    # weights streamed per stage
    (1, 2048, 5, 5, 512, "u8", "u8", True, False, "upward"),    # 16 streamed k-blocks
]


@pytest.mark.parametrize("cfg", TRANS_CASES, ids=lambda c: f"C{c[1]}_K{c[4]}_{c[2]}x{c[3]}_{c[9]}")
def test_wide_pointwise_channel_major(cfg):
    N, C, H, W, K, adt, odt, relu, act6, mode = cfg
    case = gen.conv_case(1600 + C + K, N, C, H, W, K, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), 1, adt, "s8",
                         out_dtype=odt, relu=relu, act6=act6, rounding=mode)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), mismatch_report(got, want)


@pytest.mark.parametrize("mink", ["64", "128"], ids=["channel_major", "pixel_major"])
def test_pointwise_k64_channel_major_subprocess(mink):
    """K_out = 64 pointwise: on the channel-major kernel as half a channel block (the default,
    QNN_TRANS_MINK=64) and on the pixel-major kernel (QNN_TRANS_MINK=128)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
from gpu_helpers import gpu_conv, oracle_conv
from workloads import gen
for i, (C, adt, mode) in enumerate([(256, "u8", "upward"), (64, "s8", "tonearest")]):
    case = gen.conv_case(1750 + i, 2, C, 13, 11, 64, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), 1, adt, "s8", rounding=mode)
    _, _, y = gpu_conv(case)
    assert np.array_equal(y.cpu().numpy(), oracle_conv(case)), i
print("OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, QNN_TRANS_MINK=mink),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


def test_wide_pointwise_pixel_major_subprocess():
    """QNN_NO_TRANS=1 keeps the pixel-major kernel for the same shapes."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
from gpu_helpers import gpu_conv, oracle_conv
from workloads import gen
for i, (C, K) in enumerate([(64, 256), (256, 512)]):
    case = gen.conv_case(1700 + i, 2, C, 9, 10, K, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), 1, "u8", "s8")
    _, _, y = gpu_conv(case)
    assert np.array_equal(y.cpu().numpy(), oracle_conv(case))
print("OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, QNN_NO_TRANS="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


@pytest.mark.parametrize("sets", ["1", "2", "4"])
def test_staged_row_epilogue_sets_subprocess(sets):
    """QNN_EPI_SETS=1/2/4: the staged-row plans' epilogue warp sets on alternate tiles (4 is the
    default) -- stride-1 staged rows at BN 64 / 128 with ragged tails, plus an im2col and a
    1x1 shape that keep their own plans."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
from gpu_helpers import gpu_conv, oracle_conv
from workloads import gen
cfgs = [(4, 64, 20, 19, 64, 3, 3, (1, 1), (1, 1, 1, 1)), (3, 128, 17, 15, 128, 3, 3, (1, 1), (1, 1, 1, 1)),
        (3, 128, 17, 15, 128, 3, 3, (2, 2), (1, 1, 1, 1)), (4, 256, 14, 13, 64, 1, 1, (1, 1), (0, 0, 0, 0))]
for i, (N, C, H, W, K, R, S, st, pad) in enumerate(cfgs):
    case = gen.conv_case(1800 + i, N, C, H, W, K, R, S, st, pad, (1, 1), 1, "u8", "s8")
    _, _, y = gpu_conv(case)
    assert np.array_equal(y.cpu().numpy(), oracle_conv(case)), i
print("OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, QNN_EPI_SETS=sets),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


@pytest.mark.parametrize("cfg", [
    (2, 64, 11, 9, 64, 3, 3, (1, 1), (1, 1, 1, 1), 117),
    (2, 96, 14, 14, 300, 3, 3, (2, 2), (0, 1, 1, 0), 131),
    (1, 256, 14, 14, 256, 1, 1, (1, 1), (0, 0, 0, 0), 0),
    (1, 64, 56, 56, 64, 3, 3, (1, 1), (1, 1, 1, 1), 255),
])
def test_legalize_u8_weights_to_s8(cfg):
    """SURVEY §8f row f4, the VNNI Legalize: u8 x u8 weights re-expressed as s8 with
    zp_W - 128 by one qnn_requantize launch give the same bytes as the direct u8 x u8 lowering,
    and both equal the oracle of the original (u8 x u8) problem."""
    from paper_2006_10226_b200 import PackedConv2d
    from paper_2006_10226_b200.qnn import legalize_s8_weights
    N, C, H, W, K, R, S, st, pad, zpW = cfg
    case = gen.conv_case(7000 + K, N, C, H, W, K, R, S, st, pad, (1, 1), 1, "u8", "u8", zp_W=zpW, per_channel=False)
    want = oracle_conv(case)
    w_d = torch.from_numpy(case.W).cuda()
    w8, zp2 = legalize_s8_weights(w_d, zpW)
    torch.cuda.synchronize()
    assert w8.dtype == torch.int8 and zp2 == zpW - 128
    assert np.array_equal(w8.cpu().numpy().astype(np.int16), case.W.astype(np.int16) - 128)
    x = torch.from_numpy(case.A).cuda()
    ys = []
    for wt, zp in ((w_d, zpW), (w8, zp2)):
        op = PackedConv2d(N, H, W, C, wt, torch.from_numpy(case.bias).cuda(), case.zp_A, zp, case.s_A, case.s_W,
                          case.out_params(), case.stride, case.pad, case.dil, 1)
        ys.append(op(x).cpu().numpy())
    assert np.array_equal(ys[0], want), mismatch_report(ys[0], want)
    assert np.array_equal(ys[1], want), mismatch_report(ys[1], want)


def test_channel_major_cta_pair_subprocess():
    """QNN_PAIR=1: every channel-major layer whose channel blocks pair up runs as CTA pairs
    (cta_group::2, M = 256 over two SMs): plain, split-weight (zp_W vector) and streamed-weight
    shapes, ragged pixel tails, bit-exact against the oracle.  (By default only streamed-weight
    layers with K_out >= 512 pair up; the ResNet-50 layer4 conv1 shapes at batch 2 are one.)"""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
from gpu_helpers import gpu_conv, oracle_conv
from workloads import gen
cases = [(2, 64, 9, 7, 256, "upward"), (1, 256, 13, 11, 512, "tonearest"), (2, 2048, 7, 7, 512, "upward"),
         (1, 1024, 5, 9, 1024, "upward")]
for i, (N, C, H, W, K, mode) in enumerate(cases):
    case = gen.conv_case(1850 + i, N, C, H, W, K, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), 1, "u8", "s8", rounding=mode)
    _, _, y = gpu_conv(case)
    assert np.array_equal(y.cpu().numpy(), oracle_conv(case)), i
case = gen.conv_case(1860, 2, 128, 9, 9, 256, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), 1, "u8", "s8", relu=False)
g = np.random.default_rng(1861)
case.zp_W = g.integers(-127, 128, size=256).astype(np.int32)
case.s_out = float(np.float32(case.s_out * 2))
_, _, y = gpu_conv(case)
assert np.array_equal(y.cpu().numpy(), oracle_conv(case)), "split"
print("OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, QNN_PAIR="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


def test_pixel_major_cta_pair_subprocess():
    """QNN_PAIR=1 also turns on the pixel-major kernel's CTA-pair variants (cta_group::2: the two
    M tiles of a cluster form one M = 256 MMA, each CTA staging half of the weight tile): strided
    3x3 (im2col), stride-1 3x3, strided 1x1, BN = 192 / 256, a dense with int32 output, both
    rounding modes, ragged M tails -- bit-exact against the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "tools/pair_quick_pm.py"], cwd=root, env=dict(os.environ, QNN_PAIR="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), (r.stdout[-2000:], r.stderr[-2000:])
