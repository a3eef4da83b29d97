#!/usr/bin/env python
"""SURVEY §8f rows f2 + f3: the paper's own evaluation axis on B200.

f2 (fig:money_server): QNN-int8 vs a well-optimised floating-point
execution of the same model on the same hardware.  The floating-point arm is
torchvision's ResNet-50 (random init, eval mode, BN folded into the convs) run by PyTorch /
cuDNN in channels_last, captured as one CUDA graph, in three precisions:
fp32 (TF32 off: the paper's fp32), tf32 and bf16.  Harness only -- cuDNN is
the comparison system, not part of the product path.  The int8 arm is the
bench's full ResNet-50 forward (`GpuResNet50Full`: quantize, 53 qnn.conv2d,
max pool, 16 fused residual adds, avg pool, qnn.dense, dequantize) on this
library.  Same batch, same f32 224x224 input resident in HBM, CUDA events.

f3 (fig:memory): runtime memory footprint split into
weights (parameters) and intermediate feature maps, int8 vs fp32.  fp arms:
the CUDA caching allocator (weights = bytes allocated by the model, feature
maps = peak allocated during a forward minus weights minus the input; cuDNN
workspaces included).  int8 arm: weights = the prepacked buffers (weights,
folded offsets, multipliers); feature maps = the peak live set over one traced
forward (each buffer live from its first to its last use, i.e. what a
graph-level planner reusing dead buffers holds) plus the conv workspaces.
The analytic weight count (conv + fc weights only, no BN) comes from
`workloads.shapes` (pinned to torchvision in tests/test_shapes_cpu.py).

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


def _fold_bn(m):
    """Fold every eval-mode BatchNorm into the conv before it (what a pre-quantized int8 model has
    already done, and what an optimised fp32 deployment does), so both arms run the same math."""
    from torch.nn.utils.fusion import fuse_conv_bn_eval
    m.conv1 = fuse_conv_bn_eval(m.conv1, m.bn1)
    m.bn1 = torch.nn.Identity()
    for layer in (m.layer1, m.layer2, m.layer3, m.layer4):
        for b in layer:
            for i in (1, 2, 3):
                setattr(b, f"conv{i}", fuse_conv_bn_eval(getattr(b, f"conv{i}"), getattr(b, f"bn{i}")))
                setattr(b, f"bn{i}", torch.nn.Identity())
            if b.downsample is not None:
                b.downsample = torch.nn.Sequential(fuse_conv_bn_eval(b.downsample[0], b.downsample[1]))
    return m


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
    model = _fold_bn(torchvision.models.resnet50().eval()).to(dev, dtype=dtype).to(memory_format=torch.channels_last)
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


class _Trace:
    """Records, per library call of one forward, which storages it reads and which it writes."""

    def __init__(self):
        self.events = []     # (reads: {ptr: bytes}, writes: {ptr: bytes})

    @staticmethod
    def _tensors(obj, acc):
        if isinstance(obj, torch.Tensor):
            st = obj.untyped_storage()
            acc[st.data_ptr()] = (st.nbytes(), obj.element_size())
        elif isinstance(obj, (tuple, list)):
            for o in obj:
                _Trace._tensors(o, acc)
        return acc

    def wrap(self, fn):
        def call(*args, **kw):
            out = kw.get("out")
            reads = self._tensors([a for a in args] + [v for k, v in kw.items() if k != "out"], {})
            self.events.append((reads, self._tensors(out, {})))
            return fn(*args, **kw)
        return call

    def peak_live(self, exclude=(), as_fp32=False):
        """Peak bytes over the call sequence when each buffer lives from its first to its last use
        (what a graph-level memory planner reusing dead buffers achieves).  as_fp32: the same graph
        with every buffer holding 4-byte elements (the fp32 execution of the same call sequence)."""
        first, last, size = {}, {}, {}
        for i, (r, w) in enumerate(self.events):
            for p, b in list(r.items()) + list(w.items()):
                if p in exclude:
                    continue
                first.setdefault(p, i)
                last[p] = i
                size[p] = b[0] // b[1] * 4 if as_fp32 else b[0]
        return max(sum(size[p] for p in size if first[p] <= i <= last[p]) for i in range(len(self.events)))


class _QnnProxy:
    def __init__(self, mod, tr):
        self._mod, self._tr = mod, tr

    def __getattr__(self, name):
        f = getattr(self._mod, name)
        return self._tr.wrap(f) if name.startswith("qnn_") else f


def int8_arm(batch, steps, dev):
    import bench
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    m = bench.resnet50_full_model(batch)
    net = bench.GpuResNet50Full(m, dev)
    torch.cuda.synchronize()
    ops = list(net.ops.values()) + [net.fc]
    packed = sum(o.packed.numel() for o in ops)
    ws = sum(o.workspace.numel() for o in ops if o.workspace is not None)
    act = sum(t.numel() * t.element_size() for t in net.buf.values())
    act += sum(t.numel() * t.element_size() for t in (net.q_image, net.pool, net.gap, net.fc_out, net.logits))
    in_bytes = net.image_d.numel() * net.image_d.element_size()
    # one traced forward: buffer liveness under the real call sequence
    tr = _Trace()
    real_ops, real_fc, real_q = dict(net.ops), net.fc, net.qnn
    net.ops = {k: tr.wrap(v) for k, v in real_ops.items()}
    net.fc = tr.wrap(real_fc)
    net.qnn = _QnnProxy(real_q, tr)
    net.step()
    torch.cuda.synchronize()
    net.ops, net.fc, net.qnn = real_ops, real_fc, real_q
    ex = {net.image_d.untyped_storage().data_ptr()}
    live, live32 = tr.peak_live(exclude=ex), tr.peak_live(exclude=ex, as_fp32=True)
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
           "weights_bytes": int(packed), "workspace_bytes": int(ws), "feature_map_bytes": int(live + ws),
           "feature_map_bytes_allocated": int(act),
           "feature_map_bytes_same_graph_fp32": int(live32), "input_bytes": int(in_bytes), "library_calls": len(tr.events),
           "note": "weights = prepacked buffers (weights + folded offsets + multipliers); feature maps = peak "
                   "live set over the traced call sequence (buffers reused once dead, as a graph memory "
                   "planner does) + conv workspaces; feature_map_bytes_allocated = what the bench's "
                   "no-reuse allocation actually holds"}
    del net
    torch.cuda.empty_cache()
    return res


def analytic_weights():
    from workloads.shapes import resnet50_convs, resnet50_fc
    conv_params = sum(c.K * (c.C // c.groups) * c.R * c.S for c in resnet50_convs())
    fin, fout = resnet50_fc()
    n = conv_params + fin * fout
    bias = sum(c.K for c in resnet50_convs()) + fout
    return {"params": n, "int8_bytes": n, "fp32_bytes": 4 * (n + bias)}


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
    aw = analytic_weights()
    res["analytic_weights"] = aw
    res["footprint_int8_pct_of_fp32_same_graph"] = {
        "weights": round(100.0 * i8["weights_bytes"] / aw["fp32_bytes"], 1),
        "feature_maps": round(100.0 * i8["feature_map_bytes"] / i8["feature_map_bytes_same_graph_fp32"], 1),
        "total": round(100.0 * (i8["weights_bytes"] + i8["feature_map_bytes"]) /
                       (aw["fp32_bytes"] + i8["feature_map_bytes_same_graph_fp32"]), 1),
        "note": "fp32 side: analytic conv+fc weights (+ fp32 bias) and the int8 forward's buffer "
                "liveness with 4-byte elements; the cuDNN-measured split also counts cuDNN "
                "workspaces and the caching allocator's peak"}
    res["paper_context"] = {"speedup_vs_fp32": {"Xeon Cascade Lake": 2.35, "T4": 2.15, "Pi3": 1.35, "Pi4": 1.40},
                            "footprint_total_pct_servers": "26-33", "cite": "P:17, P:439-443, P:434"}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
