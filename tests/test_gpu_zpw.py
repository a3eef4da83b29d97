"""GPU parity for weight zero points folded into the contraction (SURVEY §8f row f4 and the
round-1 review's "zp_W != 0 on the fast path"): weights packed as W - zp_W[k] in two s8
k-block sets, so Term 3 (zp_W * sum A) is computed by the tensor cores and no row-sum
pass runs.  Per-channel zero-point vectors (reading R11 extended channel by channel) and the
per-tensor TFLite-style u8 case, on every kernel family, bit-exact against the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from gpu_helpers import gpu_conv, gpu_dense, mismatch_report, oracle_conv, oracle_dense
from workloads import gen

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# N, C, H, W, K, R, stride, pad, w dtype  -- the kernel family each shape lands on
SHAPES = [
    (2, 64, 11, 9, 64, 3, (1, 1), (1, 1, 1, 1), "s8"),      # staged-row 3x3 (resident weights)
    (2, 64, 12, 12, 96, 3, (2, 2), (1, 1, 1, 1), "u8"),     # im2col, border classes
    (2, 128, 9, 11, 256, 1, (1, 1), (0, 0, 0, 0), "s8"),    # channel-major pointwise
    (1, 256, 9, 9, 128, 1, (1, 1), (0, 0, 0, 0), "u8"),     # channel-major, K = 128
    (1, 512, 8, 8, 300, 3, (1, 1), (1, 1, 1, 1), "s8"),     # streamed weights, 2 N tiles, K tail
    (2, 96, 10, 10, 48, 1, (2, 2), (0, 0, 0, 0), "u8"),     # strided 1x1 (pixel-major)
]


def _vec_case(seed, N, C, H, W, K, R, st, pad, wdt, mode):
    case = gen.conv_case(seed, N, C, H, W, K, R, R, st, pad, (1, 1), 1, "u8", wdt, zp_W=0, rounding=mode,
                         relu=False, zp_out=128)
    g = np.random.default_rng(seed + 1)
    lo, hi = (1, 255) if wdt == "u8" else (-127, 127)
    zpv = g.integers(lo, hi + 1, size=K).astype(np.int32)
    zpv[0], zpv[-1] = lo, hi                       # the extremes of the splittable range
    case.zp_W = zpv
    case.s_out = float(np.float32(case.s_out * 2))
    return case


@pytest.mark.parametrize("i", range(len(SHAPES)))
@pytest.mark.parametrize("mode", ["upward", "tonearest"])
def test_per_channel_weight_zero_points(i, mode):
    case = _vec_case(8100 + i, *SHAPES[i], mode)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), oracle_conv(case)
    assert np.array_equal(got, want), f"{SHAPES[i]} {mode}\n" + mismatch_report(got, want)


def test_per_channel_weight_zero_points_depthwise():
    for adt in ("u8", "s8"):
        case = gen.conv_case(8150, 2, 48, 9, 10, 48, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), 48, adt, "s8", relu=False)
        case.zp_W = np.random.default_rng(8151).integers(-20, 21, size=48).astype(np.int32)
        _, _, y = gpu_conv(case)
        got, want = y.cpu().numpy(), oracle_conv(case)
        assert np.array_equal(got, want), mismatch_report(got, want)


def test_per_channel_weight_zero_points_dense():
    for wdt, lo, hi in (("s8", -127, 127), ("u8", 1, 255)):
        d = gen.dense_case(8160, 130, 384, 512, w_dtype=wdt, zp_W=0)
        d.zp_W = np.random.default_rng(8161).integers(lo, hi + 1, size=384).astype(np.int32)
        d.s_out = float(np.float32(d.s_out * 2))
        _, _, y = gpu_dense(d)
        got, want = y.cpu().numpy(), oracle_dense(d)
        assert np.array_equal(got, want), mismatch_report(got, want)


def test_unsplittable_zero_point_vector_is_rejected():
    """s8 weights with zp_W[k] = -128: W - zp_W reaches 255, outside two s8 parts."""
    from paper_2006_10226_b200 import PackedConv2d, QnnError
    case = _vec_case(8170, 1, 32, 8, 8, 32, 3, (1, 1), (1, 1, 1, 1), "s8", "upward")
    case.zp_W[3] = -128
    with pytest.raises(QnnError, match="UNSUPPORTED"):
        gpu_conv(case)


_AB = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from gpu_helpers import gpu_conv, oracle_conv
from workloads import gen
ok = True
for i, (C, K, R, st, zp) in enumerate([(64, 64, 3, 1, 121), (128, 256, 1, 1, 7), (256, 128, 3, 2, 250)]):
    c = gen.conv_case(8200 + i, 2, C, 10, 11, K, R, R, (st, st), ((R - 1) // 2,) * 4, (1, 1), 1, "u8", "u8",
                      zp_W=zp, per_channel=False)
    _, _, y = gpu_conv(c)
    ok &= bool(np.array_equal(y.cpu().numpy(), oracle_conv(c)))
print("OK" if ok else "MISMATCH")
"""


@pytest.mark.parametrize("env", [{}, {"QNN_NO_WSPLIT": "1"}], ids=["split", "row_sums"])
def test_per_tensor_zero_point_both_lowerings(env):
    """TFLite-1.13-style u8 weights with a per-tensor zp_W: the split-weight contraction
    (default) and the row-sum pass (QNN_NO_WSPLIT=1) both match the oracle."""
    code = _AB.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       env={**os.environ, **env})
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("OK"), r.stdout


@pytest.mark.parametrize("wdt,zp", [("u8", 128), ("s8", -5)])
def test_stem_zero_point_split(wdt, zp):
    """The smem-built stem (width fold) with zp_W != 0: split weights in the build-mode GEMM."""
    for K in (64, 32):
        case = gen.conv_case(8300 + K, 2, 3, 37, 37, K, 7 if K == 64 else 3, 7 if K == 64 else 3, (2, 2),
                             (3, 3, 3, 3) if K == 64 else (0, 0, 0, 0), (1, 1), 1, "u8", wdt, zp_W=zp,
                             per_channel=False, relu=True)
        _, _, y = gpu_conv(case)
        got, want = y.cpu().numpy(), oracle_conv(case)
        assert np.array_equal(got, want), mismatch_report(got, want)
