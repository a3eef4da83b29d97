"""Seeded synthetic tensors (numpy PCG64 via ``default_rng``).

Values are uniform over the full dtype range (never constant or zero) so that
both the oracle and the kernels see realistic data.
Nothing here implements the method; ``calibrated_out_scale`` only picks an
output scale from the *input statistics* (uniform-distribution moments) so
requantized outputs use the dtype range instead of saturating.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_RANGE = {"s8": (-128, 127), "u8": (0, 255)}
_NP = {"s8": np.int8, "u8": np.uint8}


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def rand_q(g: np.random.Generator, shape, dtype: str, lo=None, hi=None) -> np.ndarray:
    a, b = _RANGE[dtype]
    a = a if lo is None else lo
    b = b if hi is None else hi
    return g.integers(a, b + 1, size=shape, dtype=np.int64).astype(_NP[dtype])


def _uniform_var(lo: int, hi: int, zp: int) -> float:
    """E[(X - zp)^2] for X ~ U{lo..hi} (input statistics only)."""
    n = hi - lo + 1
    mean = (lo + hi) / 2.0
    var = (n * n - 1) / 12.0
    return var + (mean - zp) ** 2


def calibrated_out_scale(kk: int, a_range, zp_A: int, w_range, zp_W: int, s_A: float, s_W: float,
                         out_levels: float = 255.0, sigmas: float = 6.0) -> float:
    """s_out such that +-sigmas standard deviations of the real-valued output span ``out_levels``."""
    sd = math.sqrt(kk * _uniform_var(*a_range, zp_A) * _uniform_var(*w_range, zp_W))
    return float(np.float32(sigmas * sd * s_A * s_W / out_levels))


def calibrated_out_scale_var(kk: int, var_a: float, var_w: float, s_A: float, s_W: float,
                             out_levels: float = 255.0, sigmas: float = 6.0) -> float:
    """As calibrated_out_scale, from the second moments of the zero-point-subtracted input and
    weight codes (e.g. a post-ReLU activation calibrated to 6 sigma over 255 levels has
    E[a^2] = (255/6)^2 / 2 ~ 903, not the uniform distribution's ~21675)."""
    sd = math.sqrt(kk * var_a * var_w)
    return float(np.float32(sigmas * sd * s_A * s_W / out_levels))


POST_RELU_VAR = (255.0 / 6.0) ** 2 / 2.0      # E[y^2] of max(0, N(0, s)) coded at 6 s / 255 per level


@dataclass
class ConvCase:
    """One qnn.conv2d problem in the kernels' NHWC / OHWI layout."""
    A: np.ndarray            # N,H,W,C (u8/s8)
    W: np.ndarray            # K,R,S,C/G (s8/u8)
    bias: np.ndarray | None  # K int32
    zp_A: int
    zp_W: int
    s_A: float
    s_W: np.ndarray          # 1 or K float32
    s_out: float
    zp_out: int
    out_dtype: str
    stride: tuple
    pad: tuple
    dil: tuple
    groups: int
    relu: bool
    act_min: int | None = None
    act_max: int | None = None
    rounding: str = "upward"

    @property
    def a_dtype(self):
        return "u8" if self.A.dtype == np.uint8 else "s8"

    @property
    def w_dtype(self):
        return "u8" if self.W.dtype == np.uint8 else "s8"

    def nchw(self):
        return np.ascontiguousarray(self.A.transpose(0, 3, 1, 2))

    def oihw(self):
        return np.ascontiguousarray(self.W.transpose(0, 3, 1, 2))

    def out_params(self):
        if self.out_dtype == "s32":
            return None
        return dict(scale=self.s_out, zero_point=self.zp_out, dtype=self.out_dtype,
                    rounding=self.rounding, relu=self.relu, act_min=self.act_min, act_max=self.act_max)


def conv_case(seed: int, N: int, C: int, H: int, W: int, K: int, R: int, S: int,
              stride=(1, 1), pad=(0, 0, 0, 0), dil=(1, 1), groups: int = 1,
              a_dtype="u8", w_dtype="s8", zp_A=None, zp_W=0, per_channel=True,
              out_dtype="u8", zp_out=None, relu=True, rounding="upward", bias=True,
              act6=False) -> ConvCase:
    g = rng(seed)
    A = rand_q(g, (N, H, W, C), a_dtype)
    # s8 weights over the full code range, -128 included (a symmetric TFLite-style quantizer would
    # stop at -127; the kernels must handle the extreme code regardless)
    lo_w, hi_w = _RANGE[w_dtype]
    Wt = rand_q(g, (K, R, S, C // groups), w_dtype, lo_w, hi_w)
    if zp_A is None:
        zp_A = int(g.integers(*_RANGE[a_dtype])) if a_dtype == "u8" else int(g.integers(-64, 64))
    s_A = float(np.float32(g.uniform(0.01, 0.05)))
    if per_channel:
        s_W = g.uniform(0.002, 0.02, size=K).astype(np.float32)
    else:
        s_W = np.array([g.uniform(0.002, 0.02)], np.float32)
    kk = (C // groups) * R * S
    s_out = calibrated_out_scale(kk, _RANGE[a_dtype], zp_A, (lo_w, hi_w), zp_W, s_A, float(np.median(s_W)))
    if zp_out is None:
        zp_out = 0 if relu else (128 if out_dtype == "u8" else 0)
    b = g.integers(-4096, 4097, size=K).astype(np.int32) if bias else None
    act_min = act_max = None
    if act6:
        # ReLU6: real 6.0 in the output domain (TFLite-style output clamp, reading R6)
        act_max = int(min(_RANGE.get(out_dtype, (0, 255))[1], zp_out + round(6.0 / s_out)))
    return ConvCase(A, Wt, b, zp_A, zp_W, s_A, s_W, s_out, zp_out, out_dtype, tuple(stride), tuple(pad),
                    tuple(dil), groups, relu, None, act_max, rounding)


@dataclass
class DenseCase:
    A: np.ndarray      # M,K
    W: np.ndarray      # N,K
    bias: np.ndarray | None
    zp_A: int
    zp_W: int
    s_A: float
    s_W: np.ndarray
    s_out: float
    zp_out: int
    out_dtype: str
    relu: bool
    rounding: str = "upward"

    @property
    def a_dtype(self):
        return "u8" if self.A.dtype == np.uint8 else "s8"

    @property
    def w_dtype(self):
        return "u8" if self.W.dtype == np.uint8 else "s8"

    def out_params(self):
        if self.out_dtype == "s32":
            return None
        return dict(scale=self.s_out, zero_point=self.zp_out, dtype=self.out_dtype,
                    rounding=self.rounding, relu=self.relu)


def dense_case(seed: int, M: int, N: int, K: int, a_dtype="u8", w_dtype="s8", zp_A=None, zp_W=0,
               per_channel=True, out_dtype="u8", zp_out=None, relu=False, rounding="upward",
               bias=True) -> DenseCase:
    g = rng(seed)
    A = rand_q(g, (M, K), a_dtype)
    lo_w, hi_w = _RANGE[w_dtype]   # full code range, -128 included
    Wt = rand_q(g, (N, K), w_dtype, lo_w, hi_w)
    if zp_A is None:
        zp_A = int(g.integers(1, 255)) if a_dtype == "u8" else int(g.integers(-64, 64))
    s_A = float(np.float32(g.uniform(0.01, 0.05)))
    s_W = (g.uniform(0.002, 0.02, size=N) if per_channel else g.uniform(0.002, 0.02, size=1)).astype(np.float32)
    s_out = calibrated_out_scale(K, _RANGE[a_dtype], zp_A, (lo_w, hi_w), zp_W, s_A, float(np.median(s_W)))
    if zp_out is None:
        zp_out = 0 if relu else (128 if out_dtype == "u8" else 0)
    b = g.integers(-4096, 4097, size=N).astype(np.int32) if bias else None
    return DenseCase(A, Wt, b, zp_A, zp_W, s_A, s_W, s_out, zp_out, out_dtype, relu, rounding)
