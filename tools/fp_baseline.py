#!/usr/bin/env python
"""SURVEY §8f rows f2 + f3: the paper's own evaluation axis on B200.

f2 (fig:money_server): QNN-int8 vs a well-optimised floating-point
execution of the same model on the same hardware.  The floating-point arm is
torchvision's ResNet-50 (random init, eval mode, BN live) run by PyTorch /
cuDNN in channels_last, captured as one CUDA graph, in three precisions:
fp32 (TF32 off: the paper's fp32), tf32 and bf16.  Harness only -- cuDNN is
the comparison system, not part of the product path.  The int8 arm is the
bench's full ResNet-50 forward (`GpuResNet50Full`: quantize, 53 qnn.conv2d,
max pool, 16 fused residual adds, avg pool, qnn.dense, dequantize) on this
library.  Same batch, same f32 224x224 input resident in HBM, CUDA events.

f3 (fig:memory): runtime memory footprint split into
weights (parameters) and intermediate feature maps, int8 vs fp32.  Measured
with the CUDA caching allocator: weights = bytes allocated while building the
model (int8: packed weights + folded offsets / multipliers, before any
activation buffer), feature maps = peak allocated during a forward minus
weights minus the f32 input.  The analytic weight bytes (conv + fc weights
only, no BN) come from `workloads.shapes` for reference.

Prints one JSON line.  Usage: python tools/fp_baseline.py [--batch 256] [--steps 30]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def _time_graph(fn, steps, warmup=3):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warmup):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, g


def fp_arm(mode, batch, steps, dev):
    import torchvision
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = mode == "tf32"
    torch.backends.cuda.matmul.allow_tf32 = mode == "tf32"
    dtype = torch.bfloat16 if mode == "bf16" else torch.float32
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.manual_seed(0)
    model = torchvision.models.resnet50().eval().to(dev, dtype=dtype).to(memory_format=torch.channels_last)
    torch.cuda.synchronize()
    w_bytes = torch.cuda.memory_allocated() - base
    x = torch.randn(batch, 3, 224, 224, device=dev).contiguous(memory_format=torch.channels_last)
    in_bytes = x.numel() * x.element_size()
    out = {}

    def fwd():
        with torch.inference_mode():
            out["y"] = model(x.to(dtype)).float()

    torch.cuda.reset_peak_memory_stats()
    fwd()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    ms, g = _time_graph(fwd, steps)
    del g, model, x, out
    torch.cuda.empty_cache()
    return {"images_per_s": round(batch / (ms / 1000.0), 1), "ms_per_step": round(ms, 4),
            "weights_bytes": int(w_bytes), "feature_map_bytes": int(peak - w_bytes - in_bytes),
            "input_bytes": int(in_bytes)}


def int8_arm(batch, steps, dev):
    import bench
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    m = bench.resnet50_full_model(batch)
    net = bench.GpuResNet50Full(m, dev)
    torch.cuda.synchronize()
    total_static = torch.cuda.memory_allocated() - base
    # weights = packed per-layer state (everything the ops own); buffers are the activations
    act = sum(t.numel() * t.element_size() for t in net.buf.values())
    act += sum(t.numel() * t.element_size() for t in (net.q_image, net.pool, net.gap, net.fc_out, net.logits))
    in_bytes = net.image_d.numel() * net.image_d.element_size()
    w_bytes = total_static - act - in_bytes
    torch.cuda.reset_peak_memory_stats()
    net.step()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    net.capture()
    for _ in range(3):
        net.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        net.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    res = {"images_per_s": round(batch / (ms / 1000.0), 1), "ms_per_step": round(ms, 4),
           "weights_bytes": int(w_bytes), "feature_map_bytes": int(peak - w_bytes - in_bytes),
           "feature_map_bytes_allocated": int(act), "input_bytes": int(in_bytes),
           "note": "every intermediate buffer is allocated separately (no reuse), so feature maps are "
                   "the sum over all layers, not the peak live set"}
    del net
    torch.cuda.empty_cache()
    return res


def analytic_weights():
    from workloads.shapes import resnet50_convs, resnet50_fc
    conv_params = sum(c.K * (c.C // c.groups) * c.R * c.S for c in resnet50_convs())
    fin, fout = resnet50_fc()
    n = conv_params + fin * fout
    return {"params": n, "int8_bytes": n, "fp32_bytes": 4 * n}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--modes", default="fp32,tf32,bf16")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    res = {"workload": f"ResNet-50 224x224 batch {args.batch}, f32 input resident in HBM, CUDA graph replay",
           "int8": int8_arm(args.batch, args.steps, dev)}
    for mode in args.modes.split(","):
        res[mode] = fp_arm(mode, args.batch, args.steps, dev)
    i8 = res["int8"]
    res["speedup_int8_vs"] = {m: round(i8["images_per_s"] / res[m]["images_per_s"], 3)
                              for m in args.modes.split(",")}
    if "fp32" in res:
        f = res["fp32"]
        res["footprint_int8_pct_of_fp32"] = {
            "weights": round(100.0 * i8["weights_bytes"] / f["weights_bytes"], 1),
            "feature_maps": round(100.0 * i8["feature_map_bytes"] / max(1, f["feature_map_bytes"]), 1),
            "total": round(100.0 * (i8["weights_bytes"] + i8["feature_map_bytes"]) /
                           (f["weights_bytes"] + f["feature_map_bytes"]), 1)}
    res["analytic_weights"] = analytic_weights()
    res["paper_context"] = {"speedup_vs_fp32": {"Xeon Cascade Lake": 2.35, "T4": 2.15, "Pi3": 1.35, "Pi4": 1.40},
                            "footprint_total_pct_servers": "26-33", "cite": "P:17, P:439-443, P:434"}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
