"""Thin Python binding of libqnn.so (include/qnn.h) — argument marshalling only.

Every step of the path runs in the CUDA kernels behind the C ABI; PyTorch only
provides device memory (``data_ptr()``) and the current CUDA stream.  There is
no CPU fallback: if ``libqnn.so`` is missing or a call fails, an exception is
raised.  Function names mirror the C entry points.
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import Sequence

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# QNN_LIB: load an alternative in-tree build (A/B experiments); defaults to the package's libqnn.so
LIB_PATH = os.environ.get("QNN_LIB") or os.path.join(_PKG, "libqnn.so")
_lock = threading.Lock()
_lib = None

QNN_S8, QNN_U8, QNN_S32, QNN_F32 = 0, 1, 2, 3
ROUNDING = {"upward": 0, "tonearest": 1}
STATUS = {0: "QNN_OK", 1: "QNN_ERR_INVALID_VALUE", 2: "QNN_ERR_UNSUPPORTED", 3: "QNN_ERR_MISALIGNED",
          4: "QNN_ERR_WORKSPACE", 5: "QNN_ERR_CUDA"}
_TORCH_DT = {torch.int8: QNN_S8, torch.uint8: QNN_U8, torch.int32: QNN_S32, torch.float32: QNN_F32}
_DT_TORCH = {v: k for k, v in _TORCH_DT.items()}
_NAME_DT = {"s8": QNN_S8, "u8": QNN_U8, "s32": QNN_S32, "f32": QNN_F32}
INT32_MIN, INT32_MAX = -(2 ** 31), 2 ** 31 - 1

EXPORTED = ["qnn_status_string", "qnn_launch_counter", "qnn_launch_counter_reset", "qnn_derive_multiplier",
            "qnn_conv2d_prepack_size", "qnn_conv2d_prepack", "qnn_conv2d_workspace_size", "qnn_conv2d_packed",
            "qnn_conv2d", "qnn_depthwise_conv2d", "qnn_dense_prepack_size", "qnn_dense_prepack",
            "qnn_dense_workspace_size", "qnn_dense_packed", "qnn_dense", "qnn_requantize", "qnn_quantize",
            "qnn_dequantize", "qnn_add", "qnn_pool2d", "qnn_conv2d_packed_add", "qnn_quantize_host",
            "qnn_dequantize_host"]


class QnnError(RuntimeError):
    pass


class Pool2dDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("N", "H", "W", "C", "R", "S", "stride_h", "stride_w", "pad_t",
                                               "pad_l", "pad_b", "pad_r", "in_cstride", "out_cstride")] + \
               [("dtype", ctypes.c_int), ("mode", ctypes.c_int)]


class OutputParams(ctypes.Structure):
    _fields_ = [("output_scale", ctypes.c_float), ("output_zero_point", ctypes.c_int32),
                ("out_dtype", ctypes.c_int), ("rounding", ctypes.c_int), ("relu", ctypes.c_int32),
                ("act_min", ctypes.c_int32), ("act_max", ctypes.c_int32)]


class Conv2dDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("N", "H", "W", "C", "K", "R", "S", "stride_h", "stride_w", "pad_t", "pad_l", "pad_b", "pad_r",
                 "dil_h", "dil_w", "groups", "in_cstride", "out_cstride")] + [
        ("input_dtype", ctypes.c_int), ("kernel_dtype", ctypes.c_int),
        ("input_zero_point", ctypes.c_int32), ("kernel_zero_point", ctypes.c_int32),
        ("input_scale", ctypes.c_float), ("kernel_scales", ctypes.POINTER(ctypes.c_float)),
        ("num_kernel_scales", ctypes.c_int32), ("kernel_zero_points", ctypes.POINTER(ctypes.c_int32)),
        ("num_kernel_zero_points", ctypes.c_int32)]


class DenseDesc(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("N", ctypes.c_int32), ("K", ctypes.c_int32), ("lda", ctypes.c_int32),
                ("ldc", ctypes.c_int32), ("a_dtype", ctypes.c_int), ("w_dtype", ctypes.c_int),
                ("zp_A", ctypes.c_int32), ("zp_W", ctypes.c_int32), ("s_A", ctypes.c_float),
                ("s_W", ctypes.POINTER(ctypes.c_float)), ("n_sW", ctypes.c_int32),
                ("zp_Ws", ctypes.POINTER(ctypes.c_int32)), ("n_zpW", ctypes.c_int32)]


def lib() -> ctypes.CDLL:
    """Load libqnn.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                if os.environ.get("QNN_AUTOBUILD"):
                    from . import build as _b
                    _b.build()
                else:
                    raise QnnError(f"{LIB_PATH} not built; run `python -m paper_2006_10226_b200.build`")
            L = ctypes.CDLL(LIB_PATH)
            vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
            cdp, odp, ddp = ctypes.POINTER(Conv2dDesc), ctypes.POINTER(OutputParams), ctypes.POINTER(DenseDesc)
            L.qnn_status_string.restype = ctypes.c_char_p
            L.qnn_launch_counter.restype = ctypes.c_uint64
            L.qnn_derive_multiplier.argtypes = [ctypes.c_double, ctypes.POINTER(i32), ctypes.POINTER(i32)]
            L.qnn_conv2d_prepack_size.argtypes = [cdp, odp, ctypes.POINTER(sz)]
            L.qnn_conv2d_prepack.argtypes = [cdp, vp, vp, odp, vp, sz, vp]
            L.qnn_conv2d_workspace_size.argtypes = [cdp, odp, ctypes.POINTER(sz)]
            L.qnn_conv2d_packed.argtypes = [cdp, odp, vp, vp, vp, vp, sz, vp]
            L.qnn_conv2d.argtypes = [cdp, vp, vp, vp, odp, vp, vp, sz, vp]
            L.qnn_depthwise_conv2d.argtypes = [cdp, vp, vp, vp, odp, vp, vp, sz, vp]
            L.qnn_dense_prepack_size.argtypes = [ddp, odp, ctypes.POINTER(sz)]
            L.qnn_dense_prepack.argtypes = [ddp, vp, vp, odp, vp, sz, vp]
            L.qnn_dense_workspace_size.argtypes = [ddp, odp, ctypes.POINTER(sz)]
            L.qnn_dense_packed.argtypes = [ddp, odp, vp, vp, vp, vp, sz, vp]
            L.qnn_dense.argtypes = [ddp, vp, vp, vp, odp, vp, vp, sz, vp]
            L.qnn_requantize.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int, ctypes.POINTER(i64), i32, i32,
                                         ctypes.POINTER(ctypes.c_float), i32, i32, ctypes.c_float, i32,
                                         ctypes.c_int, vp]
            L.qnn_quantize.argtypes = [vp, vp, ctypes.c_int, ctypes.POINTER(i64), i32, i32,
                                       ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32), i32, vp]
            L.qnn_dequantize.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(i64), i32, i32,
                                         ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32), i32, vp]
            L.qnn_quantize_host.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.POINTER(i64), i32, i32,
                                            ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32), i32, vp, vp]
            L.qnn_dequantize_host.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(i64), i32, i32,
                                              ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32), i32, vp]
            f32 = ctypes.c_float
            L.qnn_add.argtypes = [vp, ctypes.c_int, f32, i32, vp, ctypes.c_int, f32, i32, vp, ctypes.c_int, f32, i32,
                                  i64, ctypes.c_int, i32, vp]
            L.qnn_pool2d.argtypes = [ctypes.POINTER(Pool2dDesc), vp, vp, vp]
            L.qnn_conv2d_packed_add.argtypes = [cdp, odp, vp, vp, vp, ctypes.c_int, f32, i32, i32, vp, vp, sz, vp]
            for name in EXPORTED:
                if name not in ("qnn_status_string", "qnn_launch_counter", "qnn_launch_counter_reset"):
                    getattr(L, name).restype = ctypes.c_int
            _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        raise QnnError(f"{what}: {STATUS.get(status, status)}")


def _stream(stream=None) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev(t: torch.Tensor, name: str):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise QnnError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise QnnError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _floats(v) -> ctypes.Array:
    vals = [float(x) for x in (v.tolist() if hasattr(v, "tolist") else (v if isinstance(v, Sequence) else [v]))]
    return (ctypes.c_float * len(vals))(*vals)


def _ints(v) -> ctypes.Array:
    vals = [int(x) for x in (v.tolist() if hasattr(v, "tolist") else (v if isinstance(v, Sequence) else [v]))]
    return (ctypes.c_int32 * len(vals))(*vals)


def _dtcode(dt) -> int:
    if isinstance(dt, str):
        return _NAME_DT[dt]
    return _TORCH_DT[dt]


def launch_counter() -> int:
    return int(lib().qnn_launch_counter())


def launch_counter_reset():
    lib().qnn_launch_counter_reset()


def qnn_derive_multiplier(m: float) -> tuple[int, int]:
    M, s = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().qnn_derive_multiplier(float(m), ctypes.byref(M), ctypes.byref(s)), "qnn_derive_multiplier")
    return M.value, s.value


def output_params(scale: float, zero_point: int, dtype="u8", rounding="upward", relu=False, act_min=None,
                  act_max=None) -> OutputParams:
    return OutputParams(float(scale), int(zero_point), _dtcode(dtype), ROUNDING[rounding], int(bool(relu)),
                        INT32_MIN if act_min is None else int(act_min), INT32_MAX if act_max is None else int(act_max))


# --------------------------------------------------------------------------- conv2d / depthwise
class PackedConv2d:
    """qnn.conv2d with its compile-time folding done once.

    ``x`` NHWC (u8/s8), ``w`` OHWI (K,R,S,C/groups) on the GPU, ``bias`` int32[K] or None.
    ``out`` None -> raw int32 Eq. 3 result (+bias); else a dict (scale, zero_point, dtype,
    rounding, relu, act_min, act_max) for the fused requantize epilogue.
    """

    def __init__(self, N, H, W, C, w: torch.Tensor, bias: torch.Tensor | None, zp_A: int, zp_W: int, s_A: float,
                 s_W, out: dict | None = None, stride=(1, 1), pad=(0, 0, 0, 0), dil=(1, 1), groups=1,
                 input_dtype="u8", in_cstride=0, out_cstride=0, stream=None):
        K, R, S, Cg = w.shape
        self._scales = _floats(s_W)
        d = Conv2dDesc()
        for k, v in dict(N=N, H=H, W=W, C=C, K=K, R=R, S=S, stride_h=stride[0], stride_w=stride[1], pad_t=pad[0],
                         pad_l=pad[1], pad_b=pad[2], pad_r=pad[3], dil_h=dil[0], dil_w=dil[1], groups=groups,
                         in_cstride=in_cstride, out_cstride=out_cstride).items():
            setattr(d, k, int(v))
        d.input_dtype = _dtcode(input_dtype)
        d.kernel_dtype = _dtcode(w.dtype)
        d.input_zero_point = int(zp_A)
        if isinstance(zp_W, (int,)) or (hasattr(zp_W, "ndim") and getattr(zp_W, "ndim") == 0):
            d.kernel_zero_point = int(zp_W)
        else:   # per-channel weight zero points (f4)
            self._zps = _ints(zp_W)
            d.kernel_zero_point = 0
            d.kernel_zero_points = ctypes.cast(self._zps, ctypes.POINTER(ctypes.c_int32))
            d.num_kernel_zero_points = len(self._zps)
        d.input_scale = float(s_A)
        d.kernel_scales = ctypes.cast(self._scales, ctypes.POINTER(ctypes.c_float))
        d.num_kernel_scales = len(self._scales)
        self.desc = d
        self.out = out
        self.o = output_params(**out) if out is not None else None
        self._op = ctypes.byref(self.o) if self.o is not None else None
        self.P = (H + pad[0] + pad[2] - dil[0] * (R - 1) - 1) // stride[0] + 1
        self.Q = (W + pad[1] + pad[3] - dil[1] * (S - 1) - 1) // stride[1] + 1
        self.K = K
        self.out_dtype = _DT_TORCH[self.o.out_dtype] if self.o is not None else torch.int32
        L = lib()
        n = ctypes.c_size_t()
        _check(L.qnn_conv2d_prepack_size(ctypes.byref(d), self._op, ctypes.byref(n)), "qnn_conv2d_prepack_size")
        dev = w.device
        self.packed = torch.empty(max(n.value, 256), dtype=torch.uint8, device=dev)
        _check(L.qnn_conv2d_prepack(ctypes.byref(d), _dev(w, "w"), None if bias is None else _dev(bias, "bias"),
                                    self._op, ctypes.c_void_p(self.packed.data_ptr()), n.value,
                                    ctypes.c_void_p(_stream(stream))), "qnn_conv2d_prepack")
        _check(L.qnn_conv2d_workspace_size(ctypes.byref(d), self._op, ctypes.byref(n)), "qnn_conv2d_workspace_size")
        self.ws_bytes = n.value
        self.workspace = torch.empty(max(n.value, 256), dtype=torch.uint8, device=dev) if n.value else None

    def out_shape(self):
        d = self.desc
        return (d.N, self.P, self.Q, d.out_cstride or self.K)

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None, residual=None,
                 out_channel_offset: int = 0) -> torch.Tensor:
        """Run the conv; residual=(tensor NHWC, scale, zero_point) fuses a qnn.add of it (reading R19).
        With out_cstride set at construction, ``out`` may be a wider NHWC buffer (e.g. an Inception
        concat) and the conv writes channels [out_channel_offset, + K) of every pixel."""
        if out is None:
            out = torch.empty(self.out_shape(), dtype=self.out_dtype, device=x.device)
        optr = _dev(out, "out")
        if out_channel_offset:
            if not self.desc.out_cstride or out.shape[-1] != self.desc.out_cstride:
                raise QnnError("out_channel_offset needs out_cstride == out.shape[-1]")
            optr = ctypes.c_void_p(optr.value + int(out_channel_offset) * out.element_size())
        ws = ctypes.c_void_p(self.workspace.data_ptr()) if self.workspace is not None else None
        if residual is None:
            _check(lib().qnn_conv2d_packed(ctypes.byref(self.desc), self._op, ctypes.c_void_p(self.packed.data_ptr()),
                                           _dev(x, "x"), optr, ws, self.ws_bytes,
                                           ctypes.c_void_p(_stream(stream))), "qnn_conv2d_packed")
        else:
            r, rs, rz = residual
            _check(lib().qnn_conv2d_packed_add(ctypes.byref(self.desc), self._op,
                                               ctypes.c_void_p(self.packed.data_ptr()), _dev(x, "x"),
                                               _dev(r, "residual"), _TORCH_DT[r.dtype], float(rs), int(rz), 0,
                                               _dev(out, "out"), ws, self.ws_bytes,
                                               ctypes.c_void_p(_stream(stream))), "qnn_conv2d_packed_add")
        return out


def qnn_conv2d(x: torch.Tensor, w: torch.Tensor, bias, zp_A, zp_W, s_A, s_W, out: dict | None = None,
               stride=(1, 1), pad=(0, 0, 0, 0), dil=(1, 1), groups=1) -> torch.Tensor:
    """One-shot qnn.conv2d (prepack + run) on NHWC x / OHWI w."""
    N, H, W, C = x.shape
    op = PackedConv2d(N, H, W, C, w, bias, zp_A, zp_W, s_A, s_W, out, stride, pad, dil, groups,
                      input_dtype="s8" if x.dtype == torch.int8 else "u8")
    return op(x)


def qnn_depthwise_conv2d(x, w, bias, zp_A, zp_W, s_A, s_W, out=None, stride=(1, 1), pad=(0, 0, 0, 0), dil=(1, 1)):
    C = x.shape[3]
    return qnn_conv2d(x, w, bias, zp_A, zp_W, s_A, s_W, out, stride, pad, dil, groups=C)


# --------------------------------------------------------------------------- dense
class PackedDense:
    """qnn.dense: out[m, n] over A (M x K) and W (N x K) with folded constants."""

    def __init__(self, M, w: torch.Tensor, bias, zp_A, zp_W, s_A, s_W, out: dict | None = None, a_dtype="u8",
                 stream=None):
        N, K = w.shape
        self._scales = _floats(s_W)
        d = DenseDesc()
        d.M, d.N, d.K, d.lda, d.ldc = int(M), int(N), int(K), 0, 0
        d.a_dtype = _dtcode(a_dtype)
        d.w_dtype = _dtcode(w.dtype)
        if isinstance(zp_W, (int,)) or (hasattr(zp_W, "ndim") and getattr(zp_W, "ndim") == 0):
            d.zp_A, d.zp_W, d.s_A = int(zp_A), int(zp_W), float(s_A)
        else:   # per-channel weight zero points (f4)
            self._zps = _ints(zp_W)
            d.zp_A, d.zp_W, d.s_A = int(zp_A), 0, float(s_A)
            d.zp_Ws = ctypes.cast(self._zps, ctypes.POINTER(ctypes.c_int32))
            d.n_zpW = len(self._zps)
        d.s_W = ctypes.cast(self._scales, ctypes.POINTER(ctypes.c_float))
        d.n_sW = len(self._scales)
        self.desc = d
        self.o = output_params(**out) if out is not None else None
        self._op = ctypes.byref(self.o) if self.o is not None else None
        self.out_dtype = _DT_TORCH[self.o.out_dtype] if self.o is not None else torch.int32
        L = lib()
        n = ctypes.c_size_t()
        _check(L.qnn_dense_prepack_size(ctypes.byref(d), self._op, ctypes.byref(n)), "qnn_dense_prepack_size")
        self.packed = torch.empty(max(n.value, 256), dtype=torch.uint8, device=w.device)
        _check(L.qnn_dense_prepack(ctypes.byref(d), _dev(w, "w"), None if bias is None else _dev(bias, "bias"),
                                   self._op, ctypes.c_void_p(self.packed.data_ptr()), n.value,
                                   ctypes.c_void_p(_stream(stream))), "qnn_dense_prepack")
        _check(L.qnn_dense_workspace_size(ctypes.byref(d), self._op, ctypes.byref(n)), "qnn_dense_workspace_size")
        self.ws_bytes = n.value
        self.workspace = torch.empty(max(n.value, 256), dtype=torch.uint8, device=w.device) if n.value else None

    def __call__(self, a: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((self.desc.M, self.desc.N), dtype=self.out_dtype, device=a.device)
        ws = ctypes.c_void_p(self.workspace.data_ptr()) if self.workspace is not None else None
        _check(lib().qnn_dense_packed(ctypes.byref(self.desc), self._op, ctypes.c_void_p(self.packed.data_ptr()),
                                      _dev(a, "a"), _dev(out, "out"), ws, self.ws_bytes,
                                      ctypes.c_void_p(_stream(stream))), "qnn_dense_packed")
        return out


def qnn_dense(a: torch.Tensor, w: torch.Tensor, bias, zp_A, zp_W, s_A, s_W, out: dict | None = None):
    op = PackedDense(a.shape[0], w, bias, zp_A, zp_W, s_A, s_W, out, a_dtype="s8" if a.dtype == torch.int8 else "u8")
    return op(a)


# --------------------------------------------------------------------------- elementwise
def _shape(t: torch.Tensor):
    shp = list(t.shape) or [1]
    return (ctypes.c_int64 * len(shp))(*shp), len(shp)


def qnn_requantize(x: torch.Tensor, in_scales, in_zp: int, out_scale: float, out_zp: int, out_dtype="u8",
                   rounding="upward", axis=-1, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    odt = _dtcode(out_dtype)
    if out is None:
        out = torch.empty(x.shape, dtype=_DT_TORCH[odt], device=x.device)
    shp, nd = _shape(x)
    sc = _floats(in_scales)
    _check(lib().qnn_requantize(_dev(x, "x"), _TORCH_DT[x.dtype], _dev(out, "out"), odt, shp, nd, int(axis), sc,
                                len(sc), int(in_zp), float(out_scale), int(out_zp), ROUNDING[rounding],
                                ctypes.c_void_p(_stream(stream))), "qnn_requantize")
    return out


def legalize_s8_weights(w: torch.Tensor, zp_W: int, stream=None) -> tuple[torch.Tensor, int]:
    """QNN Legalize for u8 x u8 convs: represent the u8 weights
    as s8 by inserting a requantize before the weight operand, Q_W' = Q_W - 128, and shift the
    zero point, zp_W' = zp_W - 128.  (Q_W - zp_W) is unchanged, so Eq. 3 gives the same Q_C.
    Runs as one qnn_requantize launch (scales 1, in_zp zp_W, out_zp zp_W - 128, s8 out: exact,
    no rounding).  tcgen05 takes u8 x u8 natively, so this is the alternative lowering, not a
    requirement; the parity tests run both."""
    if w.dtype != torch.uint8:
        raise QnnError("legalize_s8_weights: weights must be u8")
    zp2 = int(zp_W) - 128
    return qnn_requantize(w, [1.0], int(zp_W), 1.0, zp2, "s8", stream=stream), zp2


def qnn_quantize(x: torch.Tensor, scales, zero_points, out_dtype="u8", axis=-1, out=None, stream=None):
    odt = _dtcode(out_dtype)
    if out is None:
        out = torch.empty(x.shape, dtype=_DT_TORCH[odt], device=x.device)
    shp, nd = _shape(x)
    sc, zp = _floats(scales), _ints(zero_points)
    if len(zp) == 1 and len(sc) > 1:
        zp = _ints([zp[0]] * len(sc))
    if len(sc) == 1 and len(zp) > 1:
        sc = _floats([sc[0]] * len(zp))
    _check(lib().qnn_quantize(_dev(x, "x"), _dev(out, "out"), odt, shp, nd, int(axis), sc, zp, len(sc),
                              ctypes.c_void_p(_stream(stream))), "qnn_quantize")
    return out


def qnn_dequantize(q: torch.Tensor, scales, zero_points, axis=-1, out=None, stream=None):
    if out is None:
        out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    shp, nd = _shape(q)
    sc, zp = _floats(scales), _ints(zero_points)
    if len(zp) == 1 and len(sc) > 1:
        zp = _ints([zp[0]] * len(sc))
    if len(sc) == 1 and len(zp) > 1:
        sc = _floats([sc[0]] * len(zp))
    _check(lib().qnn_dequantize(_dev(q, "q"), _TORCH_DT[q.dtype], _dev(out, "out"), shp, nd, int(axis), sc, zp,
                                len(sc), ctypes.c_void_p(_stream(stream))), "qnn_dequantize")
    return out


def _pinned(t: torch.Tensor, name: str):
    if not isinstance(t, torch.Tensor) or t.is_cuda or not t.is_pinned():
        raise QnnError(f"{name} must be a pinned (page-locked) host tensor")
    if not t.is_contiguous():
        raise QnnError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _params(scales, zero_points):
    sc, zp = _floats(scales), _ints(zero_points)
    if len(zp) == 1 and len(sc) > 1:
        zp = _ints([zp[0]] * len(sc))
    if len(sc) == 1 and len(zp) > 1:
        sc = _floats([sc[0]] * len(zp))
    return sc, zp


def qnn_quantize_host(x_host: torch.Tensor, staging: torch.Tensor, out: torch.Tensor, scales, zero_points,
                      out_dtype="u8", axis=-1, copy_stream=None, stream=None):
    """qnn_quantize_host: pinned host f32 -> (copy engine, copy_stream) staging -> quantize -> out
    on stream (the C-ABI entry of an end-to-end step; see include/qnn.h for the ordering rules)."""
    if staging.numel() < x_host.numel() or staging.dtype != torch.float32:
        raise QnnError("staging must be a float32 CUDA tensor at least as large as the input")
    shp, nd = _shape(x_host)
    sc, zp = _params(scales, zero_points)
    _check(lib().qnn_quantize_host(_pinned(x_host, "x_host"), _dev(staging, "staging"), _dev(out, "out"),
                                   _dtcode(out_dtype), shp, nd, int(axis), sc, zp, len(sc),
                                   ctypes.c_void_p(_stream(copy_stream)), ctypes.c_void_p(_stream(stream))),
           "qnn_quantize_host")
    return out


def qnn_dequantize_host(q: torch.Tensor, out_host: torch.Tensor, scales, zero_points, axis=-1, stream=None):
    """qnn_dequantize_host: the dequantize kernel writes straight into pinned host memory."""
    if out_host.dtype != torch.float32 or out_host.numel() != q.numel():
        raise QnnError("out_host must be a float32 tensor with q's element count")
    shp, nd = _shape(q)
    sc, zp = _params(scales, zero_points)
    _check(lib().qnn_dequantize_host(_dev(q, "q"), _TORCH_DT[q.dtype], _pinned(out_host, "out_host"), shp, nd,
                                     int(axis), sc, zp, len(sc), ctypes.c_void_p(_stream(stream))),
           "qnn_dequantize_host")
    return out_host


# --------------------------------------------------------------------------- glue
def qnn_add(a: torch.Tensor, s_a: float, zp_a: int, b: torch.Tensor, s_b: float, zp_b: int, s_out: float,
            zp_out: int, out_dtype="u8", rounding="upward", relu=False, out=None, stream=None) -> torch.Tensor:
    """qnn.add of two 8-bit tensors (same shape), requantized to (s_out, zp_out) (reading R19)."""
    if a.shape != b.shape:
        raise QnnError("qnn_add: shapes differ")
    odt = _dtcode(out_dtype)
    if out is None:
        out = torch.empty(a.shape, dtype=_DT_TORCH[odt], device=a.device)
    _check(lib().qnn_add(_dev(a, "a"), _TORCH_DT[a.dtype], float(s_a), int(zp_a), _dev(b, "b"), _TORCH_DT[b.dtype],
                         float(s_b), int(zp_b), _dev(out, "out"), odt, float(s_out), int(zp_out), a.numel(),
                         ROUNDING[rounding], int(bool(relu)), ctypes.c_void_p(_stream(stream))), "qnn_add")
    return out


def qnn_pool2d(x: torch.Tensor, mode: str, R: int, S: int, stride=(1, 1), pad=(0, 0, 0, 0), out=None,
               stream=None, out_channel_offset: int = 0) -> torch.Tensor:
    """Max / average pooling of an NHWC 8-bit tensor (padding excluded, reading R20).  ``out`` may
    be wider than x (a concat buffer): the result goes to channels [out_channel_offset, + C)."""
    N, H, W, C = x.shape
    P = (H + pad[0] + pad[2] - R) // stride[0] + 1
    Q = (W + pad[1] + pad[3] - S) // stride[1] + 1
    if out is None:
        out = torch.empty((N, P, Q, C), dtype=x.dtype, device=x.device)
    ocs = out.shape[-1] if out.shape[-1] != C or out_channel_offset else 0
    d = Pool2dDesc(N, H, W, C, R, S, stride[0], stride[1], pad[0], pad[1], pad[2], pad[3], 0, ocs,
                   _TORCH_DT[x.dtype], 0 if mode == "max" else 1)
    optr = _dev(out, "out")
    if out_channel_offset:
        optr = ctypes.c_void_p(optr.value + int(out_channel_offset) * out.element_size())
    _check(lib().qnn_pool2d(ctypes.byref(d), _dev(x, "x"), optr, ctypes.c_void_p(_stream(stream))), "qnn_pool2d")
    return out
