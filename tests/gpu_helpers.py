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
