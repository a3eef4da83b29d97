"""Shared helpers for the -m gpu parity tests: run a seeded case through the
CUDA path (C ABI via the thin binding) and through the oracle, same bytes."""
from __future__ import annotations

import numpy as np
import torch

import oracle as orc
from workloads.gen import ConvCase, DenseCase


def to_dev(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_conv(case: ConvCase, out_cstride: int = 0):
    from paper_2006_10226_b200 import PackedConv2d
    N, H, W, C = case.A.shape
    op = PackedConv2d(N, H, W, C, to_dev(case.W), to_dev(case.bias), case.zp_A, case.zp_W, case.s_A, case.s_W,
                      case.out_params(), case.stride, case.pad, case.dil, case.groups, input_dtype=case.a_dtype,
                      out_cstride=out_cstride)
    x = to_dev(case.A)
    y = op(x)
    torch.cuda.synchronize()
    return op, x, y


def oracle_conv(case: ConvCase):
    """Oracle output in NHWC (the oracle itself works in NCHW)."""
    y = orc.qnn_conv2d(case.nchw(), case.oihw(), case.zp_A, case.zp_W, case.s_A, case.s_W, case.bias,
                       case.out_params(), case.stride, case.pad, case.dil, case.groups)
    return np.ascontiguousarray(y.transpose(0, 2, 3, 1))


def oracle_conv_at(case: ConvCase, idx_nhwc: np.ndarray, P: int, Q: int):
    """Oracle values at flat NPQK indices, requantized exactly like qnn_conv2d."""
    K = case.W.shape[0]
    idx = np.asarray(idx_nhwc, np.int64)
    k = idx % K
    t = idx // K
    q = t % Q
    t //= Q
    p = t % P
    n = t // P
    nkpq = ((n * K + k) * P + p) * Q + q
    acc = orc.conv2d_acc_at(case.nchw(), case.oihw(), case.zp_A, case.zp_W, nkpq, case.bias, case.stride, case.pad,
                            case.dil, case.groups)
    o = case.out_params()
    if o is None:
        return acc.astype(np.int32)
    M, S = orc.conv_multipliers(case.s_A, case.s_W, o["scale"], K)
    Mk = M[k] if M.size > 1 else np.full(k.size, M[0], np.int32)
    Sk = S[k] if S.size > 1 else np.full(k.size, S[0], np.int32)
    out = np.empty(idx.size, np.uint8 if o["dtype"] == "u8" else np.int8)
    for i in range(idx.size):
        out[i] = orc.requantize_acc(acc[i:i + 1], Mk[i:i + 1], Sk[i:i + 1], o["dtype"], o["zero_point"],
                                    o["rounding"], o["relu"], o.get("act_min"), o.get("act_max"), axis=0)[0]
    return out


def gpu_dense(case: DenseCase):
    from paper_2006_10226_b200 import PackedDense
    op = PackedDense(case.A.shape[0], to_dev(case.W), to_dev(case.bias), case.zp_A, case.zp_W, case.s_A, case.s_W,
                     case.out_params(), a_dtype=case.a_dtype)
    a = to_dev(case.A)
    y = op(a)
    torch.cuda.synchronize()
    return op, a, y


def oracle_dense(case: DenseCase):
    return orc.qnn_dense(case.A, case.W, case.zp_A, case.zp_W, case.s_A, case.s_W, case.bias, case.out_params())


def mismatch_report(got: np.ndarray, want: np.ndarray, limit: int = 8) -> str:
    bad = np.argwhere(got != want)
    lines = [f"{bad.shape[0]} of {got.size} differ"]
    for b in bad[:limit]:
        b = tuple(b)
        lines.append(f"  at {b}: got {got[b]} want {want[b]}")
    return "\n".join(lines)


def ref_conv_lib(A_nhwc, W_ohwi, zp_A, zp_W, bias, s_A, s_W, out, stride=(1, 1), pad=(0, 0, 0, 0), dil=(1, 1),
                 groups=1, chunk=16):
    """Exact reference for FULL-SIZE layers (too large for the int64 loop oracle in a test).

    Eq. 2's integer core sum (a - zp_A)(w - zp_W) through a library routine, torch float64
    conv2d on the zero-point-subtracted operands (zero padding of a - zp_A == zp_A padding of
    a): every product and partial sum is an integer below 255^2 * 4608 < 2^53, so the
    float64 result is exact in any summation order (SURVEY §8c pins: "Term 1 / zp = 0 special
    case ... torch.nn.functional.conv2d in float64 is exact here").  Bias and the requantize
    (Eq. 5) are the oracle's own exact-rational routines.  Returns NHWC."""
    import torch.nn.functional as F
    N = A_nhwc.shape[0]
    K = W_ohwi.shape[0]
    Wd = torch.from_numpy(np.ascontiguousarray(W_ohwi.transpose(0, 3, 1, 2)).astype(np.float64) - zp_W)
    b = np.zeros(K, np.int64) if bias is None else np.asarray(bias, np.int64)
    if out is not None:
        M, S = orc.conv_multipliers(s_A, s_W, out["scale"], K)
    res = []
    for n0 in range(0, N, chunk):
        a = torch.from_numpy(np.ascontiguousarray(A_nhwc[n0:n0 + chunk].transpose(0, 3, 1, 2)).astype(np.float64)
                             - zp_A)
        a = F.pad(a, (pad[1], pad[3], pad[0], pad[2]))
        acc = F.conv2d(a, Wd, stride=tuple(stride), dilation=tuple(dil), groups=groups)
        acc = acc.numpy().astype(np.int64) + b[None, :, None, None]
        if out is None:
            y = acc.astype(np.int32)
        else:
            y = orc.requantize_acc(acc, M, S, out.get("dtype", "u8"), out.get("zero_point", 0),
                                   out.get("rounding", "upward"), out.get("relu", False), out.get("act_min"),
                                   out.get("act_max"), axis=1)
        res.append(np.ascontiguousarray(y.transpose(0, 2, 3, 1)))
    return np.concatenate(res, 0)


def ref_conv_case(case: ConvCase, chunk=16):
    return ref_conv_lib(case.A, case.W, case.zp_A, case.zp_W, case.bias, case.s_A, case.s_W, case.out_params(),
                        case.stride, case.pad, case.dil, case.groups, chunk)
