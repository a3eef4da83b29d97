"""CPU oracle for the QNN hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
(``paper_2006_10226_b200``) never imports it and shares no code with it.

The arithmetic lives in ``qnn_oracle.cpp`` (plain C++ loops, int64
accumulation, exact-rational requantize with ``__int128``); this module only
builds/loads it and marshals numpy arrays.  Layout is the paper's NCHW / OIHW
(P:178); callers permute to/from NHWC themselves.

Each function cites the passage it follows (PAPER.md line numbers "P:n",
equation numbers as in the paper).  Readings of ambiguous passages are listed
in DESIGN.md ("R1".."R18").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qnn_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# oracle-private dtype / rounding codes (mirrors qnn_oracle.cpp, not include/qnn.h)
DT = {"s8": 0, "u8": 1, "s32": 2, "f32": 3}
NP_DT = {"s8": np.int8, "u8": np.uint8, "s32": np.int32, "f32": np.float32}
ROUND = {"upward": 0, "tonearest": 1}
RANGE = {"s8": (-128, 127), "u8": (0, 255), "s32": (-(2**31), 2**31 - 1)}


def build(force: bool = False) -> str:
    """Compile qnn_oracle.cpp -> liboracle.so (g++ -O3 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c++17",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
            L.oracle_derive_multiplier.argtypes = [ctypes.c_double, ctypes.POINTER(i32), ctypes.POINTER(i32)]
            L.oracle_derive_multiplier.restype = ctypes.c_int
            L.oracle_round_fixed.argtypes = [i64, i32, i32, ctypes.c_int]
            L.oracle_round_fixed.restype = i64
            conv_args = [ctypes.c_int] * 16 + [ctypes.c_int, vp, ctypes.c_int, vp, i32, i32, vp]
            L.oracle_conv2d_acc.argtypes = conv_args + [vp]
            L.oracle_conv2d_eq3.argtypes = conv_args + [vp]
            L.oracle_conv2d_acc_at.argtypes = conv_args + [vp, i64, vp]
            L.oracle_dense_acc.argtypes = [ctypes.c_int] * 3 + [ctypes.c_int, vp, ctypes.c_int, vp, i32, i32, vp, vp]
            L.oracle_dense_acc_at.argtypes = [ctypes.c_int] * 3 + [ctypes.c_int, vp, ctypes.c_int, vp, i32, i32, vp, vp, i64, vp]
            L.oracle_conv_multipliers.argtypes = [ctypes.c_float, vp, ctypes.c_int, ctypes.c_int, ctypes.c_float, vp, vp]
            L.oracle_conv_multipliers.restype = ctypes.c_int
            L.oracle_requantize_acc.argtypes = [vp, i64, i64, ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int,
                                                i32, ctypes.c_int, i32, i32, ctypes.c_int, vp]
            L.oracle_requantize.argtypes = [vp, ctypes.c_int, i64, i64, ctypes.c_int, vp, ctypes.c_int, i32,
                                            ctypes.c_float, i32, ctypes.c_int, ctypes.c_int, vp]
            L.oracle_requantize.restype = ctypes.c_int
            L.oracle_quantize.argtypes = [vp, i64, i64, ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int, vp]
            L.oracle_dequantize.argtypes = [vp, ctypes.c_int, i64, i64, ctypes.c_int, vp, vp, ctypes.c_int, vp]
            L.oracle_num_threads.restype = ctypes.c_int
            L.oracle_set_num_threads.argtypes = [ctypes.c_int]
            f32 = ctypes.c_float
            L.oracle_add.argtypes = [vp, ctypes.c_int, f32, i32, vp, ctypes.c_int, f32, i32, i64, f32, i32,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, vp]
            L.oracle_add.restype = ctypes.c_int
            L.oracle_pool2d.argtypes = [vp] + [ctypes.c_int] * 14 + [vp]
            _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _dt_of(a: np.ndarray) -> str:
    return {np.dtype(np.int8): "s8", np.dtype(np.uint8): "u8", np.dtype(np.int32): "s32",
            np.dtype(np.float32): "f32"}[a.dtype]


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(n: int) -> None:
    """Thread count of the oracle's later OpenMP regions (timing only; results do not depend on it)."""
    lib().oracle_set_num_threads(int(n))


# --------------------------------------------------------------------------- #
# Fixed-point multiplier and rounding (Eq. 5)                           #
# --------------------------------------------------------------------------- #
def derive_multiplier(m: float) -> tuple[int, int]:
    """(M, shift) with M in [2^30, 2^31) and m ~= M * 2^(shift-31) (reading R2)."""
    M, s = ctypes.c_int32(), ctypes.c_int32()
    if lib().oracle_derive_multiplier(float(m), ctypes.byref(M), ctypes.byref(s)) != 0:
        raise ValueError(f"multiplier must be positive and finite, got {m!r}")
    return M.value, s.value


def round_fixed(x: int, M: int, shift: int, rounding: str = "upward") -> int:
    """Exact-rational R(x * M / 2^(31-shift)) (Eq. 5 through the P:281 proxy, reading R1)."""
    return lib().oracle_round_fixed(int(x), int(M), int(shift), ROUND[rounding])


def conv_multipliers(s_A: float, s_W, s_out: float, K: int):
    """m_k = (s_A * s_W[k]) / s_out in double (Eq. 2 scale s_A*s_W; reading R3)."""
    sW = np.ascontiguousarray(np.asarray(s_W, dtype=np.float32).reshape(-1))
    M = np.zeros(K, np.int32)
    S = np.zeros(K, np.int32)
    if lib().oracle_conv_multipliers(float(s_A), _p(sW), sW.size, K, float(s_out), _p(M), _p(S)) != 0:
        raise ValueError("invalid scales")
    return M, S


# --------------------------------------------------------------------------- #
# conv2d / dense (Eq. 2 direct form with zp padding)         #
# --------------------------------------------------------------------------- #
def out_hw(H, W, R, S, stride=(1, 1), pad=(0, 0, 0, 0), dil=(1, 1)):
    pt, pl, pb, pr = pad
    P = (H + pt + pb - dil[0] * (R - 1) - 1) // stride[0] + 1
    Q = (W + pl + pr - dil[1] * (S - 1) - 1) // stride[1] + 1
    return P, Q


def _conv_common(A, Wt, stride, pad, dil, groups):
    A = np.ascontiguousarray(A)
    Wt = np.ascontiguousarray(Wt)
    N, C, H, W = A.shape
    K, Cg, R, S = Wt.shape
    assert C == Cg * groups and K % groups == 0, "channel/group mismatch"
    pt, pl, pb, pr = pad
    args = [N, C, H, W, K, R, S, stride[0], stride[1], pt, pl, pb, pr, dil[0], dil[1], groups,
            DT[_dt_of(A)], _p(A), DT[_dt_of(Wt)], _p(Wt)]
    return A, Wt, args, out_hw(H, W, R, S, stride, pad, dil)


def _per_channel(zp_W):
    """A per-output-channel weight zero-point vector, or None for a scalar."""
    z = np.asarray(zp_W)
    return None if z.ndim == 0 else z.astype(np.int64).reshape(-1)


def conv2d_acc(A, Wt, zp_A, zp_W, bias=None, stride=(1, 1), pad=(0, 0, 0, 0), dil=(1, 1), groups=1):
    """int64 acc[n,k,p,q] = sum (a - zp_A)(W - zp_W) + bias[k]; a = zp_A when padded.
    zp_W may be one value per output channel k (f4): Eq. 2 then holds channel by channel, so the
    result is assembled from one scalar-zp_W evaluation per channel (for groups == C, the
    channel's own input plane)."""
    zv = _per_channel(zp_W)
    if zv is not None:
        K = Wt.shape[0]
        assert zv.size == K and groups in (1, A.shape[1])
        parts = []
        for k in range(K):
            Ak = A[:, k:k + 1] if groups > 1 else A
            bk = None if bias is None else np.asarray(bias)[k:k + 1]
            parts.append(conv2d_acc(Ak, Wt[k:k + 1], zp_A, int(zv[k]), bk, stride, pad, dil, 1))
        return np.concatenate(parts, axis=1)
    A, Wt, args, (P, Q) = _conv_common(A, Wt, stride, pad, dil, groups)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.int32)
    out = np.zeros((A.shape[0], Wt.shape[0], P, Q), np.int64)
    lib().oracle_conv2d_acc(*args, int(zp_A), int(zp_W), _p(b), _p(out))
    return out


def conv2d_acc_at(A, Wt, zp_A, zp_W, idx, bias=None, stride=(1, 1), pad=(0, 0, 0, 0), dil=(1, 1), groups=1):
    """Same as conv2d_acc, only at flat NKPQ indices ``idx``."""
    A, Wt, args, _ = _conv_common(A, Wt, stride, pad, dil, groups)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.int32)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.zeros(idx.size, np.int64)
    lib().oracle_conv2d_acc_at(*args, int(zp_A), int(zp_W), _p(b), _p(idx), idx.size, _p(out))
    return out


def conv2d_eq3(A, Wt, zp_A, zp_W, bias=None, stride=(1, 1), pad=(0, 0, 0, 0), dil=(1, 1), groups=1):
    """Eq. 3's four terms summed separately (self-test only)."""
    A, Wt, args, (P, Q) = _conv_common(A, Wt, stride, pad, dil, groups)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.int32)
    out = np.zeros((A.shape[0], Wt.shape[0], P, Q), np.int64)
    lib().oracle_conv2d_eq3(*args, int(zp_A), int(zp_W), _p(b), _p(out))
    return out


def dense_acc(A, Wt, zp_A, zp_W, bias=None):
    """int64 acc[m,n] = sum_k (A[m,k] - zp_A)(W[n,k] - zp_W) + bias[n] (zp_W scalar or per n)."""
    zv = _per_channel(zp_W)
    if zv is not None:
        return np.concatenate([dense_acc(A, Wt[n:n + 1], zp_A, int(zv[n]),
                                         None if bias is None else np.asarray(bias)[n:n + 1])
                               for n in range(Wt.shape[0])], axis=1)
    A = np.ascontiguousarray(A)
    Wt = np.ascontiguousarray(Wt)
    M, K = A.shape
    N, K2 = Wt.shape
    assert K == K2
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.int32)
    out = np.zeros((M, N), np.int64)
    lib().oracle_dense_acc(M, N, K, DT[_dt_of(A)], _p(A), DT[_dt_of(Wt)], _p(Wt),
                           int(zp_A), int(zp_W), _p(b), _p(out))
    return out


def dense_acc_at(A, Wt, zp_A, zp_W, idx, bias=None):
    A = np.ascontiguousarray(A)
    Wt = np.ascontiguousarray(Wt)
    M, K = A.shape
    N = Wt.shape[0]
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.int32)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.zeros(idx.size, np.int64)
    lib().oracle_dense_acc_at(M, N, K, DT[_dt_of(A)], _p(A), DT[_dt_of(Wt)], _p(Wt),
                              int(zp_A), int(zp_W), _p(b), _p(idx), idx.size, _p(out))
    return out


# --------------------------------------------------------------------------- #
# Requantize (Eq. 5)                                                #
# --------------------------------------------------------------------------- #
def requantize_acc(acc, M, shift, out_dtype="u8", zp_out=0, rounding="upward", relu=False,
                   act_min=None, act_max=None, axis=1):
    """Requantize an int64 accumulator tensor: clamp(zp_out + R(relu(acc)*M_c*2^(shift_c-31)))."""
    acc = np.ascontiguousarray(acc, dtype=np.int64)
    M = np.ascontiguousarray(M, dtype=np.int32).reshape(-1)
    S = np.ascontiguousarray(shift, dtype=np.int32).reshape(-1)
    axis = axis % acc.ndim
    Cext = acc.shape[axis]
    inner = int(np.prod(acc.shape[axis + 1:], dtype=np.int64))
    assert M.size in (1, Cext)
    lo = -(2**31) if act_min is None else int(act_min)
    hi = 2**31 - 1 if act_max is None else int(act_max)
    out = np.zeros(acc.shape, NP_DT[out_dtype])
    lib().oracle_requantize_acc(_p(acc), acc.size, inner, Cext, _p(M), _p(S), M.size, ROUND[rounding],
                                int(zp_out), int(bool(relu)), lo, hi, DT[out_dtype], _p(out))
    return out


def requantize(x, in_scales, in_zp, out_scale, out_zp, out_dtype="u8", rounding="upward", axis=-1):
    """Standalone qnn.requantize: Q_B = clamp(R((s_A[c]/s_B)(Q_A - zp_A)) + zp_B) (Eq. 5)."""
    x = np.ascontiguousarray(x)
    sc = np.ascontiguousarray(np.asarray(in_scales, np.float32).reshape(-1))
    axis = axis % x.ndim
    Cext = x.shape[axis] if x.ndim else 1
    inner = int(np.prod(x.shape[axis + 1:], dtype=np.int64))
    out = np.zeros(x.shape, NP_DT[out_dtype])
    rc = lib().oracle_requantize(_p(x), DT[_dt_of(x)], x.size, inner, Cext, _p(sc), sc.size, int(in_zp),
                                 float(out_scale), int(out_zp), ROUND[rounding], DT[out_dtype], _p(out))
    if rc != 0:
        raise ValueError("invalid requantize scales")
    return out


# --------------------------------------------------------------------------- #
# Quantize / dequantize (Eq. 1)                                       #
# --------------------------------------------------------------------------- #
def _axis_params(x, axis, scales, zps):
    sc = np.ascontiguousarray(np.asarray(scales, np.float32).reshape(-1))
    zp = np.ascontiguousarray(np.asarray(zps, np.int32).reshape(-1))
    if zp.size == 1 and sc.size > 1:
        zp = np.full(sc.size, zp[0], np.int32)
    if sc.size == 1 and zp.size > 1:
        sc = np.full(zp.size, sc[0], np.float32)
    axis = axis % x.ndim
    return sc, zp, x.shape[axis], int(np.prod(x.shape[axis + 1:], dtype=np.int64))


def quantize(x, scales, zps, out_dtype="u8", axis=-1):
    """q = clamp(round_half_away(fl32(x / s)) + zp) (Eq. 1 inverted; reading R14)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    sc, zp, Cext, inner = _axis_params(x, axis, scales, zps)
    out = np.zeros(x.shape, NP_DT[out_dtype])
    lib().oracle_quantize(_p(x), x.size, inner, Cext, _p(sc), _p(zp), sc.size, DT[out_dtype], _p(out))
    return out


def dequantize(q, scales, zps, axis=-1):
    """x = fl32(s * (q - zp)) with a single rounding (Eq. 1)."""
    q = np.ascontiguousarray(q)
    sc, zp, Cext, inner = _axis_params(q, axis, scales, zps)
    out = np.zeros(q.shape, np.float32)
    lib().oracle_dequantize(_p(q), DT[_dt_of(q)], q.size, inner, Cext, _p(sc), _p(zp), sc.size, _p(out))
    return out


# --------------------------------------------------------------------------- #
# Composite: the fused conv/dense operator's expected output                  #
# --------------------------------------------------------------------------- #
def qnn_conv2d(A, Wt, zp_A, zp_W, s_A, s_W, bias=None, out=None, stride=(1, 1), pad=(0, 0, 0, 0),
               dil=(1, 1), groups=1):
    """TFLite-style qnn.conv2d -> bias_add -> clip -> qnn.requantize (fig:tflite_conv2d).

    ``out`` is None (raw int32 Eq. 3 result + bias) or a dict with keys
    scale, zero_point, dtype, rounding, relu, act_min, act_max.
    """
    acc = conv2d_acc(A, Wt, zp_A, zp_W, bias, stride, pad, dil, groups)
    return _finish(acc, s_A, s_W, out, axis=1)


def qnn_dense(A, Wt, zp_A, zp_W, s_A, s_W, bias=None, out=None):
    acc = dense_acc(A, Wt, zp_A, zp_W, bias)
    return _finish(acc, s_A, s_W, out, axis=1)


def _finish(acc, s_A, s_W, out, axis):
    if out is None:
        lo, hi = RANGE["s32"]
        assert acc.min(initial=0) >= lo and acc.max(initial=0) <= hi, "int32 overflow (reading R10)"
        return acc.astype(np.int32)
    K = acc.shape[axis]
    M, S = conv_multipliers(s_A, s_W, out["scale"], K)
    return requantize_acc(acc, M, S, out.get("dtype", "u8"), out.get("zero_point", 0),
                          out.get("rounding", "upward"), out.get("relu", False),
                          out.get("act_min"), out.get("act_max"), axis=axis)


# --------------------------------------------------------------------------- #
# Inter-layer glue: qnn.add, pooling, conv + residual add   #
# --------------------------------------------------------------------------- #
def add(a, s_a, zp_a, b, s_b, zp_b, s_out, zp_out, out_dtype="u8", rounding="upward", relu=False):
    """qnn.add: clamp(zp_out + R((a - zp_a) s_a/s_out) + R((b - zp_b) s_b/s_out)) (reading R19)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape
    out = np.zeros(a.shape, NP_DT[out_dtype])
    rc = lib().oracle_add(_p(a), DT[_dt_of(a)], ctypes.c_float(s_a), int(zp_a), _p(b), DT[_dt_of(b)],
                          ctypes.c_float(s_b), int(zp_b), a.size, ctypes.c_float(s_out), int(zp_out),
                          ROUND[rounding], int(bool(relu)), DT[out_dtype], _p(out))
    if rc != 0:
        raise ValueError("invalid add scales")
    return out


def pool2d(x, mode, R, S, stride=(1, 1), pad=(0, 0, 0, 0)):
    """Max / average pooling on quantized NCHW values (readings R17, R20)."""
    x = np.ascontiguousarray(x)
    N, C, H, W = x.shape
    P, Q = out_hw(H, W, R, S, stride, pad)
    out = np.zeros((N, C, P, Q), x.dtype)
    lib().oracle_pool2d(_p(x), DT[_dt_of(x)], int(mode == "avg"), N, C, H, W, R, S, stride[0], stride[1],
                        pad[0], pad[1], P, Q, _p(out))
    return out


def qnn_conv2d_add(A, Wt, zp_A, zp_W, s_A, s_W, bias, res, s_res, zp_res, out, stride=(1, 1),
                   pad=(0, 0, 0, 0), dil=(1, 1), groups=1):
    """qnn.conv2d whose int32 result, requantized to (s_out, 0), is added to a residual input
    requantized the same way (qnn.add of the conv's int32 output and the residual, then ReLU /
    clamps): y = clamp(zp_out + R(acc * m_k) + R((res - zp_res) * s_res / s_out)).  NCHW."""
    acc = conv2d_acc(A, Wt, zp_A, zp_W, bias, stride, pad, dil, groups)
    K = Wt.shape[0]
    M, S = conv_multipliers(s_A, s_W, out["scale"], K)
    rnd = out.get("rounding", "upward")
    y = requantize_acc(acc, M, S, "s32", 0, rnd, axis=1).astype(np.int64)
    y += requantize(np.ascontiguousarray(res), [s_res], zp_res, out["scale"], 0, "s32", rnd).astype(np.int64)
    y += int(out.get("zero_point", 0))
    zp_out = int(out.get("zero_point", 0))
    lo, hi = RANGE[out.get("dtype", "u8")]
    if out.get("relu", False):
        lo = max(lo, zp_out)
    if out.get("act_min") is not None:
        lo = max(lo, int(out["act_min"]))
    if out.get("act_max") is not None:
        hi = min(hi, int(out["act_max"]))
    return np.clip(y, lo, hi).astype(NP_DT[out.get("dtype", "u8")])
