"""GPU parity at the FULL sizes of BASELINE.json's configs, every output compared.

* configs[4]: the exact ResNet-50 batch-256 stack that ``bench.py`` times (same builder,
  same prepacked plans, same CUDA-graph-free launch sequence): the quantized image, every
  one of the 53 conv outputs, the fc's raw int32 logits and the dequantized logits, each
  checked against a reference fed the GPU's own layer input.
* configs[1]: all 23 distinct ResNet-50 conv shapes at batch 64, per-channel (s8 weights)
  and per-tensor (TFLite-1.13 style u8 weights with zp_W != 0), every output.
* configs[2]: every distinct non-depthwise MobileNet-v2 conv at batch 128, every output.

References: the oracle's own int64 loop (oracle/qnn_oracle.cpp) is exact but too slow for
~10^12 MACs in a test, so full-size outputs use gpu_helpers.ref_conv_lib: the integer core
through torch's float64 conv2d (exact: every partial sum is an integer < 2^53) plus the
oracle's exact-rational requantize; that reference is itself pinned to the int64 oracle on
CPU (tests/test_refs_cpu.py), and the first and last image of every benched layer are also
compared with the int64 oracle directly.
"""
import zlib

import numpy as np
import pytest
import torch

import oracle as orc
from gpu_helpers import gpu_conv, mismatch_report, oracle_conv, ref_conv_case, ref_conv_lib
from workloads import gen
from workloads.shapes import mobilenet_v2_convs, resnet50_unique

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _nchw(t):
    return np.ascontiguousarray(t.transpose(0, 3, 1, 2))


@pytest.fixture(scope="module")
def bench_net():
    import bench
    model = bench.resnet50_model(256)
    net = bench.GpuResNet50(model, torch.device("cuda", 0))
    net.step()
    torch.cuda.synchronize()
    return model, net


def test_bench_stack_b256_quantize_and_fc(bench_net):
    model, net = bench_net
    q = net.q_image.cpu().numpy()
    want = orc.quantize(model["image"], [model["img_scale"]], [model["img_zp"]], "u8")
    assert np.array_equal(q, want), mismatch_report(q, want)
    fc = model["fc"]
    acc = net.fc_out.cpu().numpy()
    want_acc = orc.qnn_dense(fc["A"], fc["W"], fc["zp_A"], 0, fc["s_A"], fc["s_W"], fc["bias"], None)
    assert np.array_equal(acc, want_acc), mismatch_report(acc, want_acc)
    logits = net.logits.cpu().numpy()
    want_l = orc.dequantize(want_acc, net.logit_scale, [0], axis=-1)
    # int32 input: fl32(s * fl32(q - zp)) rounds twice; BJ:north_star allows 1 ulp for dequantize
    ulps = np.abs(logits.view(np.int32).astype(np.int64) - want_l.view(np.int32).astype(np.int64))
    assert ulps.max() <= 1


@pytest.mark.parametrize("li", range(53))
def test_bench_stack_b256_every_layer(bench_net, li):
    """Layer li of the benched batch-256 step: all N*P*Q*K outputs vs the reference fed the
    GPU's own input of that layer; images 0 and 255 also vs the int64 oracle."""
    model, net = bench_net
    sp = net.stack.specs[li]
    x = net.stack.inputs[sp.name].cpu().numpy()
    got = net.stack.outs[sp.name].cpu().numpy()
    W = model["weights"][sp.name]
    bias = model["biases"][sp.name]
    want = ref_conv_lib(x, W, sp.zp_A, sp.zp_W, bias, sp.s_A, sp.s_W, sp.out, sp.stride, sp.pad)
    assert got.shape == want.shape
    assert np.array_equal(got, want), sp.name + "\n" + mismatch_report(got, want)
    for n in (0, x.shape[0] - 1):
        y = orc.qnn_conv2d(_nchw(x[n:n + 1]), _nchw(W), sp.zp_A, sp.zp_W, sp.s_A, sp.s_W, bias, sp.out, sp.stride,
                           sp.pad)
        assert np.array_equal(got[n:n + 1], y.transpose(0, 2, 3, 1)), f"{sp.name} image {n} vs int64 oracle"


@pytest.mark.parametrize("layer", resnet50_unique(), ids=lambda c: c.name)
@pytest.mark.parametrize("per_channel", [True, False], ids=["per_channel", "per_tensor"])
def test_resnet50_layers_batch64_full(layer, per_channel):
    wdt, zpW = ("s8", 0) if per_channel else ("u8", 128 + (zlib.crc32(layer.name.encode()) % 29) - 14)
    case = gen.conv_case(2000 + zlib.crc32(layer.name.encode()) % 1000, 64, layer.C, layer.H, layer.W, layer.K,
                         layer.R, layer.S, layer.stride, layer.pad, (1, 1), 1, "u8", wdt, zp_W=zpW,
                         per_channel=per_channel, relu=layer.relu)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), ref_conv_case(case)
    assert np.array_equal(got, want), layer.name + "\n" + mismatch_report(got, want)


@pytest.mark.parametrize("layer", resnet50_unique(), ids=lambda c: c.name)
def test_resnet50_layers_batch1_per_tensor_full(layer):
    """configs[1] at batch 1, per-tensor u8 weights (zp_W != 0: Term 3), int64 oracle."""
    zpW = 128 + (zlib.crc32(layer.name.encode()) % 31) - 15
    for mode in ("upward", "tonearest"):
        case = gen.conv_case(2500 + zlib.crc32(layer.name.encode()) % 1000, 1, layer.C, layer.H, layer.W, layer.K,
                             layer.R, layer.S, layer.stride, layer.pad, (1, 1), 1, "u8", "u8", zp_W=zpW,
                             per_channel=False, relu=layer.relu, rounding=mode)
        _, _, y = gpu_conv(case)
        got, want = y.cpu().numpy(), oracle_conv(case)
        assert np.array_equal(got, want), f"{layer.name} {mode}\n" + mismatch_report(got, want)


def _mobilenet_dense_unique():
    out, seen = [], set()
    for c in mobilenet_v2_convs():
        k = (c.C, c.K, c.H, c.W, c.R, c.S, c.stride, c.act6, c.relu)
        if c.groups == 1 and k not in seen:
            seen.add(k)
            out.append(c)
    return out


@pytest.mark.parametrize("layer", _mobilenet_dense_unique(), ids=lambda c: c.name)
def test_mobilenet_v2_pointwise_batch128_full(layer):
    case = gen.conv_case(5000 + zlib.crc32(layer.name.encode()) % 1000, 128, layer.C, layer.H, layer.W, layer.K,
                         layer.R, layer.S, layer.stride, layer.pad, (1, 1), 1, "u8", "s8", relu=layer.relu,
                         act6=layer.act6)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), ref_conv_case(case)
    assert np.array_equal(got, want), layer.name + "\n" + mismatch_report(got, want)


def _dw_layers():
    out, seen = [], set()
    for c in mobilenet_v2_convs():
        if c.groups > 1 and (c.C, c.stride) not in seen:
            seen.add((c.C, c.stride))
            out.append(c)
    return out


@pytest.mark.parametrize("layer", _dw_layers(), ids=lambda c: f"{c.name}_C{c.C}_s{c.stride[0]}")
def test_mobilenet_v2_depthwise_batch128_full(layer):
    case = gen.conv_case(3000 + layer.C, 128, layer.C, layer.H, layer.W, layer.K, 3, 3, layer.stride, layer.pad,
                         (1, 1), layer.C, "u8", "s8", relu=True, act6=True)
    _, _, y = gpu_conv(case)
    got, want = y.cpu().numpy(), ref_conv_case(case)
    assert np.array_equal(got, want), layer.name + "\n" + mismatch_report(got, want)
