"""GPU parity of the host-buffer entry points (the e2e path of bench.py): qnn_quantize_host
(pinned f32 host tensor -> copy engine -> staging -> quantize) and qnn_dequantize_host (the
kernel writes f32 straight into pinned host memory) against the oracle's quantize /
dequantize (Eq. 1, reading R14), with the copy on a second stream; pageable host memory is
rejected (QNN_ERR_INVALID_VALUE)."""
import numpy as np
import pytest
import torch

import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,axis,per_channel", [((2, 37, 41, 3), -1, False), ((5, 7, 1000), -1, True),
                                                    ((1,), 0, False), ((3, 130), 1, True)])
def test_quantize_host_matches_oracle(shape, axis, per_channel):
    from paper_2006_10226_b200 import qnn_quantize_host
    g = np.random.default_rng(sum(shape))
    x = (g.standard_normal(shape) * 3).astype(np.float32)
    x.reshape(-1)[:3] = [np.nan, 1e30, -1e30][:min(3, x.size)]
    C = shape[axis]
    sc = (g.uniform(0.01, 0.05, size=C if per_channel else 1)).astype(np.float32)
    zp = g.integers(0, 256, size=C if per_channel else 1).astype(np.int32)
    host = torch.from_numpy(x).pin_memory()
    staging = torch.empty(x.size, dtype=torch.float32, device="cuda")
    out = torch.empty(shape, dtype=torch.uint8, device="cuda")
    cs = torch.cuda.Stream()
    qnn_quantize_host(host, staging, out, sc, zp, "u8", axis=axis, copy_stream=cs)
    got = out.cpu().numpy()
    want = orc.quantize(x, sc, zp, "u8", axis=axis)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dt", ["s32", "u8", "s8"])
def test_dequantize_host_matches_oracle(dt):
    from paper_2006_10226_b200 import qnn_dequantize_host
    g = np.random.default_rng(3)
    lo, hi = {"s32": (-2 ** 31, 2 ** 31 - 1), "u8": (0, 255), "s8": (-128, 127)}[dt]
    npdt = {"s32": np.int32, "u8": np.uint8, "s8": np.int8}[dt]
    q = g.integers(lo, hi, size=(64, 1000), endpoint=True).astype(npdt)
    sc = g.uniform(1e-4, 1e-2, size=1000).astype(np.float32)
    zp = np.zeros(1000, np.int32) if dt == "s32" else g.integers(lo, hi + 1, size=1000).astype(np.int32)
    host_out = torch.full((64, 1000), np.nan, dtype=torch.float32).pin_memory()
    qnn_dequantize_host(torch.from_numpy(q).cuda(), host_out, sc, zp, axis=-1)
    torch.cuda.synchronize()
    want = orc.dequantize(q, sc, zp, axis=-1)
    got = host_out.numpy()
    ulps = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
    # s32: fl32(s * fl32(q - zp)) rounds twice (BJ:north_star allows 1 ulp); 8-bit inputs are exact
    assert ulps.max() <= (1 if dt == "s32" else 0)


def test_pageable_host_memory_is_rejected():
    from paper_2006_10226_b200 import QnnError, lib
    from paper_2006_10226_b200.qnn import _shape, _floats, _ints
    import ctypes
    x = torch.zeros(1024, dtype=torch.float32)          # pageable
    staging = torch.empty(1024, dtype=torch.float32, device="cuda")
    out = torch.empty(1024, dtype=torch.uint8, device="cuda")
    shp, nd = _shape(x)
    st = lib().qnn_quantize_host(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(staging.data_ptr()),
                                 ctypes.c_void_p(out.data_ptr()), 1, shp, nd, -1, _floats([0.1]), _ints([0]), 1,
                                 None, None)
    assert st == 1                                       # QNN_ERR_INVALID_VALUE
    st = lib().qnn_dequantize_host(ctypes.c_void_p(out.data_ptr()), 1, ctypes.c_void_p(x.data_ptr()), shp, nd, -1,
                                   _floats([0.1]), _ints([0]), 1, None)
    assert st == 1
    with pytest.raises(QnnError):
        from paper_2006_10226_b200 import qnn_quantize_host
        qnn_quantize_host(x, staging, out, [0.1], [0])


def test_e2e_step_logits_match_device_step():
    """bench.py's e2e step (qnn_quantize_host + graph ending in qnn_dequantize_host) gives the
    same logits, on the host, as the device-resident step, at batch 4."""
    import bench
    from paper_2006_10226_b200 import qnn_quantize_host
    m = bench.resnet50_model(4)
    net = bench.GpuResNet50(m, torch.device("cuda"))
    net.step()
    torch.cuda.synchronize()
    want = net.logits.cpu()
    host_in = torch.from_numpy(m["image"]).pin_memory()
    host_out = torch.full(tuple(want.shape), np.nan, dtype=torch.float32).pin_memory()
    net.capture_e2e(host_out)
    staging = torch.empty_like(net.image_d)
    net.q_image.zero_()
    qnn_quantize_host(host_in, staging, net.q_image, [m["img_scale"]], [m["img_zp"]], "u8",
                      copy_stream=torch.cuda.Stream())
    net.graph_e2e.replay()
    torch.cuda.synchronize()
    assert torch.equal(host_out, want)
