"""Pin of the full-size test reference (tests/gpu_helpers.ref_conv_lib: torch float64 conv
of the zero-point-subtracted operands + the oracle's exact requantize) to the int64 loop
oracle, on CPU, over the shape space the full-size GPU tests use: strides, asymmetric and
zero-point padding, dilation, groups, u8/s8 operands, zp_W != 0, raw int32 and clamps."""
import numpy as np
import pytest

from gpu_helpers import oracle_conv, ref_conv_case
from workloads import gen

CASES = [
    (2, 16, 9, 11, 24, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), 1, "u8", "s8", 0, "u8"),
    (1, 32, 12, 12, 40, 3, 3, (2, 2), (0, 1, 1, 0), (1, 1), 1, "u8", "u8", 131, "u8"),
    (2, 24, 10, 10, 24, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), 24, "u8", "s8", 0, "u8"),
    (1, 3, 30, 30, 16, 7, 7, (2, 2), (3, 3, 3, 3), (1, 1), 1, "u8", "s8", 0, "u8"),
    (1, 16, 11, 11, 16, 3, 3, (1, 1), (2, 2, 2, 2), (2, 2), 1, "s8", "s8", -3, "s8"),
    (3, 64, 7, 7, 32, 1, 1, (1, 1), (0, 0, 0, 0), (1, 1), 1, "u8", "s8", 0, "s32"),
    (1, 48, 9, 9, 48, 1, 7, (1, 1), (0, 3, 0, 3), (1, 1), 1, "u8", "s8", 0, "u8"),
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_ref_conv_lib_equals_int64_oracle(i):
    N, C, H, W, K, R, S, st, pad, dil, groups, adt, wdt, zpW, odt = CASES[i]
    for mode, act6 in (("upward", False), ("tonearest", True)):
        case = gen.conv_case(8800 + i, N, C, H, W, K, R, S, st, pad, dil, groups, adt, wdt, zp_W=zpW,
                             per_channel=wdt == "s8", out_dtype=odt, relu=i % 2 == 0, rounding=mode,
                             act6=act6 and odt == "u8")
        got = ref_conv_case(case, chunk=2)
        want = oracle_conv(case)
        assert got.dtype == want.dtype and np.array_equal(got, want), (CASES[i], mode)
