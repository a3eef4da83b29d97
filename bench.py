#!/usr/bin/env python
"""bench.py — ResNet-50 int8 images/sec on the QNN hot path (BASELINE.json metric,
configs[4]: full ResNet-50 pre-quantized int8 conv stack, synthetic weights).

One step = one pass of the whole hot path over one batch (per GPU):
  qnn_quantize (f32 image -> u8, Eq. 1)  ->  53 x qnn_conv2d (tcgen05 implicit
  GEMM, folded zero-point terms, fused requantize + ReLU, Eq. 3 + Eq. 5)  ->
  qnn_dense fc (raw int32)  ->  qnn_dequantize (logits -> f32).
Glue ops that are not on the path (max pool, residual add, global avg pool)
are not run; layers fed by them read persistent synthetic buffers.

Contract: ``python bench.py --gpus N --steps K --warmup W``.  configs[4] is a batch of 256
images SHARDED over the N GPUs (strong scaling: rank r takes images shard_range(256, r, N),
weights replicated, no collective on the data path; time = max over ranks).  Without
torchrun, ``--gpus N > 1`` launches the N ranks itself (torch.distributed.run, 127.0.0.1).
For N > 1 the line also carries a weak-scaling figure (256 images per GPU).  Rank 0 prints
ONE JSON line.  ``--impl reference`` times the CPU oracle (the reference arm of this tier)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "int8 conv TOPS (% of int8 TC peak) and ResNet-50 int8 images/sec at 1/2/4/8 B200"
WORKLOAD = "configs[4]: ResNet-50 pre-quantized int8 conv stack (53 qnn.conv2d + qnn.dense fc), synthetic weights"


# ----------------------------------------------------------------------------- model
def resnet50_model(batch: int, seed: int = 4000):
    """Synthetic pre-quantized ResNet-50: layer specs + numpy weights/biases/fresh inputs.

    Recipe: u8 activations (zp from the producer, 0 after
    ReLU, 128 otherwise), s8 symmetric per-channel weights U[-127,127] whose
    scales s_W = U(0.5, 1.5) / unit keep the real activation scale ~constant,
    int32 bias U[-4096,4096], output scale calibrated from input statistics,
    UPWARD rounding, seed 4000 + layer index.
    """
    from paper_2006_10226_b200.stack import LayerSpec
    from workloads import gen
    from workloads.shapes import resnet50_convs, resnet50_fc

    specs, weights, biases, fresh = [], {}, {}, {}
    out_q = {}      # layer name -> (zp_out, s_out)
    img_scale, img_zp = float(np.float32(4.77 / 255)), 128
    for li, c in enumerate(resnet50_convs()):
        g = gen.rng(seed + li)
        if c.name == "conv1":
            zp_A, s_A = img_zp, img_scale
        elif c.src:
            zp_A, s_A = out_q[c.src]
        else:
            zp_A, s_A = 0, 0.02
            fresh[c.name] = gen.rand_q(g, (batch, c.H, c.W, c.C), "u8")
        W = gen.rand_q(g, (c.K, c.R, c.S, c.C), "s8", -127, 127)
        kk = c.C * c.R * c.S
        # weight scales normalised so the real-valued activation scale stays ~constant
        # through the chain (the role batch-norm folding plays in a trained network)
        unit = gen.calibrated_out_scale(kk, (0, 255), zp_A, (-127, 127), 0, 1.0, 1.0)
        s_W = (g.uniform(0.5, 1.5, size=c.K) / unit).astype(np.float32)
        bias = g.integers(-4096, 4097, size=c.K).astype(np.int32)
        s_out = gen.calibrated_out_scale(kk, (0, 255), zp_A, (-127, 127), 0, s_A, float(np.median(s_W)))
        zp_out = 0 if c.relu else 128
        out = dict(scale=s_out, zero_point=zp_out, dtype="u8", rounding="upward", relu=c.relu)
        out_q[c.name] = (zp_out, s_out)
        specs.append(LayerSpec(c.name, batch, c.H, c.W, c.C, c.K, c.R, c.S, c.stride, c.pad, 1, zp_A, s_A, 0,
                               s_W, out, c.src))
        weights[c.name] = W
        biases[c.name] = bias
    fin, fout = resnet50_fc()
    g = gen.rng(seed + 99)
    fc = dict(name="fc", zp_A=0, s_A=0.02, W=gen.rand_q(g, (fout, fin), "s8", -127, 127),
              s_W=g.uniform(0.002, 0.02, size=fout).astype(np.float32),
              bias=g.integers(-4096, 4097, size=fout).astype(np.int32),
              A=gen.rand_q(g, (batch, fin), "u8"))
    image = gen.rng(seed + 98).standard_normal((batch, 224, 224, 3)).astype(np.float32)
    return dict(specs=specs, weights=weights, biases=biases, fresh=fresh, fc=fc, image=image,
                img_scale=img_scale, img_zp=img_zp)


def shard_model(model, lo: int, hi: int):
    """Rank's slice [lo, hi) of a batch built by resnet50_model (images are
    independent; weights, biases and scales are shared, every per-image array is sliced), so
    the ranks' outputs concatenate to the 1-GPU output of the same global batch."""
    from dataclasses import replace
    n = hi - lo
    fc = dict(model["fc"])
    fc["A"] = model["fc"]["A"][lo:hi]
    return dict(model, specs=[replace(sp, N=n) for sp in model["specs"]],
                fresh={k: v[lo:hi] for k, v in model["fresh"].items()}, fc=fc, image=model["image"][lo:hi])


class GpuResNet50:
    def __init__(self, model, device):
        import torch

        from paper_2006_10226_b200 import qnn
        from paper_2006_10226_b200.stack import ConvStack
        self.torch = torch
        self.qnn = qnn
        dev = device
        self.model = model
        self.image_d = torch.from_numpy(model["image"]).to(dev)
        self.q_image = torch.empty(self.image_d.shape, dtype=torch.uint8, device=dev)
        fresh = {k: torch.from_numpy(v).to(dev) for k, v in model["fresh"].items()}
        fresh["conv1"] = self.q_image
        self.stack = ConvStack(model["specs"], {k: torch.from_numpy(v).to(dev) for k, v in model["weights"].items()},
                               {k: torch.from_numpy(v).to(dev) for k, v in model["biases"].items()}, fresh, dev)
        fc = model["fc"]
        self.fc_in = torch.from_numpy(fc["A"]).to(dev)
        self.fc = qnn.PackedDense(fc["A"].shape[0], torch.from_numpy(fc["W"]).to(dev),
                                  torch.from_numpy(fc["bias"]).to(dev), fc["zp_A"], 0, fc["s_A"], fc["s_W"], None)
        self.fc_out = torch.empty((fc["A"].shape[0], fc["W"].shape[0]), dtype=torch.int32, device=dev)
        self.logit_scale = (np.float32(fc["s_A"]) * fc["s_W"].astype(np.float32)).astype(np.float32)
        self.logits = torch.empty(self.fc_out.shape, dtype=torch.float32, device=dev)
        self.graph = None

    def step(self, events=None):
        q = self.qnn
        m = self.model
        q.qnn_quantize(self.image_d, [m["img_scale"]], [m["img_zp"]], "u8", out=self.q_image)
        self.stack.run(events=events)
        self.fc(self.fc_in, out=self.fc_out)
        q.qnn_dequantize(self.fc_out, self.logit_scale, [0], axis=-1, out=self.logits)

    def capture(self):
        torch = self.torch
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.step()          # warm the attribute caches outside capture
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        self.qnn.launch_counter_reset()
        with torch.cuda.graph(self.graph):
            self.step()
        self.launches_per_step = self.qnn.launch_counter()
        torch.cuda.synchronize()

    def replay(self):
        self.graph.replay()

    def capture_e2e(self, host_out):
        """The step minus its quantize, with the logits dequantized straight into the pinned host
        buffer `host_out` (qnn_dequantize_host): the graph an end-to-end step replays after
        qnn_quantize_host has brought its image in."""
        torch, q = self.torch, self.qnn
        self.graph_e2e = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph_e2e):
            self.stack.run()
            self.fc(self.fc_in, out=self.fc_out)
            q.qnn_dequantize_host(self.fc_out, host_out, self.logit_scale, [0], axis=-1)
        torch.cuda.synchronize()


# ----------------------------------------------------------------------------- full network (f1)
def resnet50_full_model(batch: int, seed: int = 5000, fused: bool = True):
    """Synthetic pre-quantized ResNet-50 as a true forward: the 53 convs of
    resnet50_model's recipe plus the glue between them -- stem max pool, the 16 residual
    qnn.add (+ ReLU), global average pool -- feeding the fc.  Add outputs use zp 0 (post-ReLU)
    and scale 1.2 x the larger input scale.  fused: each residual add runs inside the block's
    conv3 epilogue (qnn_conv2d_packed_add: conv3 requantized straight to the add's output
    scale); else conv3 writes u8 and a separate qnn.add follows."""
    from workloads import gen
    from workloads.shapes import resnet50_convs, resnet50_fc
    img_scale, img_zp = float(np.float32(4.77 / 255)), 128
    convs, q = {}, {}
    for li, c in enumerate(resnet50_convs()):
        convs[c.name] = c
    layers = {}

    def conv(name, zp_A, s_A, li):
        c = convs[name]
        g = gen.rng(seed + li)
        W = gen.rand_q(g, (c.K, c.R, c.S, c.C), "s8", -127, 127)
        kk = c.C * c.R * c.S
        unit = gen.calibrated_out_scale(kk, (0, 255), zp_A, (-127, 127), 0, 1.0, 1.0)
        s_W = (g.uniform(0.5, 1.5, size=c.K) / unit).astype(np.float32)
        bias = g.integers(-4096, 4097, size=c.K).astype(np.int32)
        s_out = gen.calibrated_out_scale(kk, (0, 255), zp_A, (-127, 127), 0, s_A, float(np.median(s_W)))
        zp_out = 0 if c.relu else 128
        layers[name] = dict(c=c, W=W, bias=bias, zp_A=zp_A, s_A=s_A, s_W=s_W,
                            out=dict(scale=s_out, zero_point=zp_out, dtype="u8", rounding="upward", relu=c.relu))
        return zp_out, s_out

    li = 0
    zp, s = conv("conv1", img_zp, img_scale, li)
    blocks = []
    x_q = (zp, s)       # max pool keeps the quantization
    for name in [n for n in convs if n.endswith(".conv1") and n.startswith("layer")]:
        pre = name[:-len(".conv1")]
        li += 1
        c1 = conv(pre + ".conv1", x_q[0], x_q[1], li)
        li += 1
        c2 = conv(pre + ".conv2", c1[0], c1[1], li)
        li += 1
        c3 = conv(pre + ".conv3", c2[0], c2[1], li)
        sc = x_q
        if pre + ".downsample" in convs:
            li += 1
            sc = conv(pre + ".downsample", x_q[0], x_q[1], li)
        s_y = float(np.float32(1.2 * max(c3[1], sc[1])))
        if fused:
            layers[pre + ".conv3"]["out"] = dict(scale=s_y, zero_point=0, dtype="u8", rounding="upward", relu=True)
        blocks.append(dict(name=pre, sc=sc, c3=c3, y=(0, s_y), down=pre + ".downsample" in convs, fused=fused))
        x_q = (0, s_y)
    fin, fout = resnet50_fc()
    g = gen.rng(seed + 99)
    fc = dict(zp_A=x_q[0], s_A=x_q[1], W=gen.rand_q(g, (fout, fin), "s8", -127, 127),
              s_W=g.uniform(0.002, 0.02, size=fout).astype(np.float32),
              bias=g.integers(-4096, 4097, size=fout).astype(np.int32))
    image = gen.rng(seed + 98).standard_normal((batch, 224, 224, 3)).astype(np.float32)
    return dict(layers=layers, blocks=blocks, fc=fc, image=image, img_scale=img_scale, img_zp=img_zp, batch=batch)


def shard_full_model(m, lo: int, hi: int):
    return dict(m, image=m["image"][lo:hi], batch=hi - lo)


class GpuResNet50Full:
    """The full forward on the library's ops, captured as one CUDA graph."""

    def __init__(self, m, dev):
        import torch

        from paper_2006_10226_b200 import qnn
        self.torch, self.qnn, self.m = torch, qnn, m
        B = m["batch"]
        self.ops, self.buf = {}, {}
        for name, L in m["layers"].items():
            c = L["c"]
            op = qnn.PackedConv2d(B, c.H, c.W, c.C, torch.from_numpy(L["W"]).to(dev), torch.from_numpy(L["bias"]).to(dev),
                                  L["zp_A"], 0, L["s_A"], L["s_W"], L["out"], c.stride, c.pad, (1, 1), 1)
            self.ops[name] = op
            self.buf[name] = torch.empty(op.out_shape(), dtype=op.out_dtype, device=dev)
        self.image_d = torch.from_numpy(m["image"]).to(dev)
        self.q_image = torch.empty(self.image_d.shape, dtype=torch.uint8, device=dev)
        self.pool = torch.empty((B, 56, 56, 64), dtype=torch.uint8, device=dev)
        for b in m["blocks"]:
            self.buf[b["name"] + ".out"] = torch.empty_like(self.buf[b["name"] + ".conv3"])
        self.gap = torch.empty((B, 1, 1, 2048), dtype=torch.uint8, device=dev)
        fc = m["fc"]
        self.fc = qnn.PackedDense(B, torch.from_numpy(fc["W"]).to(dev), torch.from_numpy(fc["bias"]).to(dev),
                                  fc["zp_A"], 0, fc["s_A"], fc["s_W"], None)
        self.fc_out = torch.empty((B, fc["W"].shape[0]), dtype=torch.int32, device=dev)
        self.logit_scale = (np.float32(fc["s_A"]) * fc["s_W"].astype(np.float32)).astype(np.float32)
        self.logits = torch.empty(self.fc_out.shape, dtype=torch.float32, device=dev)
        self.graph = None

    def step(self):
        q, m = self.qnn, self.m
        q.qnn_quantize(self.image_d, [m["img_scale"]], [m["img_zp"]], "u8", out=self.q_image)
        self.ops["conv1"](self.q_image, out=self.buf["conv1"])
        q.qnn_pool2d(self.buf["conv1"], "max", 3, 3, (2, 2), (1, 1, 1, 1), out=self.pool)
        x = self.pool
        for b in m["blocks"]:
            n = b["name"]
            self.ops[n + ".conv1"](x, out=self.buf[n + ".conv1"])
            self.ops[n + ".conv2"](self.buf[n + ".conv1"], out=self.buf[n + ".conv2"])
            sc = x
            if b["down"]:
                self.ops[n + ".downsample"](x, out=self.buf[n + ".downsample"])
                sc = self.buf[n + ".downsample"]
            c3q, scq, yq = b["c3"], b["sc"], b["y"]
            if b["fused"]:
                self.ops[n + ".conv3"](self.buf[n + ".conv2"], out=self.buf[n + ".out"],
                                       residual=(sc, scq[1], scq[0]))
            else:
                self.ops[n + ".conv3"](self.buf[n + ".conv2"], out=self.buf[n + ".conv3"])
                q.qnn_add(self.buf[n + ".conv3"], c3q[1], c3q[0], sc, scq[1], scq[0], yq[1], yq[0], "u8", "upward",
                          relu=True, out=self.buf[n + ".out"])
            x = self.buf[n + ".out"]
        q.qnn_pool2d(x, "avg", 7, 7, out=self.gap)
        self.fc(self.gap.view(self.gap.shape[0], -1), out=self.fc_out)
        q.qnn_dequantize(self.fc_out, self.logit_scale, [0], axis=-1, out=self.logits)

    def capture(self):
        torch = self.torch
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        self.qnn.launch_counter_reset()
        with torch.cuda.graph(self.graph):
            self.step()
        self.launches_per_step = self.qnn.launch_counter()
        torch.cuda.synchronize()

    def replay(self):
        self.graph.replay()


# ----------------------------------------------------------------------------- Inception-v3 (configs[4])
def inception_v3_full_model(batch: int, seed: int = 7000):
    """Synthetic pre-quantized Inception-v3 forward (torchvision layout, 299x299), the second
    network of configs[4]: the 94 convs of workloads.shapes.inception_v3_convs with the glue
    between them -- stem max pools, per-block branches whose last convs write straight into
    their channel slice of the block's concat buffer (out_cstride; no concat op), 3x3/s1/p1
    average pools (padding excluded, reading R20) before the pool-branch 1x1s, 3x3/s2 max
    pools in the reduction blocks, the 8x8 global average pool, fc (raw int32), dequantize.

    Quantization: u8 activations, zp 0 after ReLU (the image: zp 128); every branch of a block
    requantizes to the block's output scale so the concat needs no requantize (the median of
    its branch-final convs' calibrated scales; the input scale in the reduction blocks, whose
    max-pool branch passes its input through).  Weights s8 per-channel with the ResNet recipe."""
    from workloads import gen
    from workloads.shapes import inception_v3_convs
    convs = {c.name: c for c in inception_v3_convs()}
    img_scale, img_zp = float(np.float32(4.77 / 255)), 128
    T = {"image": dict(H=299, W=299, C=3, zp=img_zp, s=img_scale)}
    layers, ops = {}, []
    counter = [0]

    # second moments of the input codes: the image (N(0,1) at 4.77/255 per level: ~53 codes RMS
    # around zp 128) or a post-ReLU activation calibrated to 6 sigma (gen.POST_RELU_VAR); the
    # uniform-input calibration of the ResNet recipe would shrink the signal ~5x per layer here
    VAR_W = ((127 + 127 + 1) ** 2 - 1) / 12.0

    def var_in(zp_A):
        return (1.0 / (4.77 / 255.0)) ** 2 if zp_A == img_zp else gen.POST_RELU_VAR

    def calib(name, zp_A, s_A):
        c = convs[name]
        g = gen.rng(seed + counter[0])
        counter[0] += 1
        kk = c.C * c.R * c.S
        unit = gen.calibrated_out_scale_var(kk, var_in(zp_A), VAR_W, 1.0, 1.0)
        W = gen.rand_q(g, (c.K, c.R, c.S, c.C), "s8", -127, 127)
        s_W = (g.uniform(0.5, 1.5, size=c.K) / unit).astype(np.float32)
        bias = g.integers(-4096, 4097, size=c.K).astype(np.int32)
        s_out = gen.calibrated_out_scale_var(kk, var_in(zp_A), VAR_W, s_A, float(np.median(s_W)))
        return W, s_W, bias, s_out

    def conv(name, src, dst=None, off=0, s_out=None):
        c = convs[name]
        t = T[src]
        assert (c.C, c.H, c.W) == (t["C"], t["H"], t["W"]), (name, c, t)
        W, s_W, bias, s_nat = calib(name, t["zp"], t["s"])
        so = float(np.float32(s_out if s_out is not None else s_nat))
        layers[name] = dict(c=c, W=W, bias=bias, zp_A=t["zp"], s_A=t["s"], s_W=s_W,
                            out=dict(scale=so, zero_point=0, dtype="u8", rounding="upward", relu=True))
        if dst is None:
            dst = name
            T[dst] = dict(H=c.P, W=c.Q, C=c.K, zp=0, s=so)
        ops.append(dict(kind="conv", name=name, src=src, dst=dst, off=off))
        return dst

    def pool(kind, src, dst, R, stride, pad, off=0, C_total=None):
        t = T[src]
        P = (t["H"] + 2 * pad - R) // stride + 1
        Q = (t["W"] + 2 * pad - R) // stride + 1
        if dst not in T:
            T[dst] = dict(H=P, W=Q, C=C_total or t["C"], zp=t["zp"], s=t["s"])
        ops.append(dict(kind=kind, src=src, dst=dst, R=R, stride=stride, pad=pad, off=off))
        return dst

    def block_scale(names, src):
        return float(np.median([calib_peek(n, T[src]) for n in names]))

    def calib_peek(name, t):
        # (the natural output scale of a conv of this shape on a post-ReLU input of scale t["s"])
        return t["s"]

    x = conv("Conv2d_1a_3x3", "image")
    x = conv("Conv2d_2a_3x3", x)
    x = conv("Conv2d_2b_3x3", x)
    x = pool("max", x, "pool1", 3, 2, 0)
    x = conv("Conv2d_3b_1x1", x)
    x = conv("Conv2d_4a_3x3", x)
    x = pool("max", x, "pool2", 3, 2, 0)

    def mixed_a(n, x, pool_features):
        t = T[x]
        ctot = 64 + 64 + 96 + pool_features
        sb = float(np.float32(block_scale([f"{n}.branch1x1", f"{n}.branch5x5_2", f"{n}.branch3x3dbl_3"], x)))
        T[n] = dict(H=t["H"], W=t["W"], C=ctot, zp=0, s=sb)
        conv(f"{n}.branch1x1", x, n, 0, sb)
        y = conv(f"{n}.branch5x5_1", x)
        conv(f"{n}.branch5x5_2", y, n, 64, sb)
        y = conv(f"{n}.branch3x3dbl_1", x)
        y = conv(f"{n}.branch3x3dbl_2", y)
        conv(f"{n}.branch3x3dbl_3", y, n, 128, sb)
        y = pool("avg", x, f"{n}.pool", 3, 1, 1)
        conv(f"{n}.branch_pool", y, n, 224, sb)
        return n

    x = mixed_a("Mixed_5b", x, 32)
    x = mixed_a("Mixed_5c", x, 64)
    x = mixed_a("Mixed_5d", x, 64)
    # Mixed_6a: the max-pool branch passes its input quantization through
    t = T[x]
    n = "Mixed_6a"
    sb = t["s"]
    T[n] = dict(H=17, W=17, C=768, zp=0, s=sb)
    conv(f"{n}.branch3x3", x, n, 0, sb)
    y = conv(f"{n}.branch3x3dbl_1", x)
    y = conv(f"{n}.branch3x3dbl_2", y)
    conv(f"{n}.branch3x3dbl_3", y, n, 384, sb)
    pool("max", x, n, 3, 2, 0, off=480)
    x = n

    def mixed_c(n, x):
        t = T[x]
        sb = float(np.float32(block_scale([f"{n}.branch1x1", f"{n}.branch7x7_3", f"{n}.branch7x7dbl_5"], x)))
        T[n] = dict(H=t["H"], W=t["W"], C=768, zp=0, s=sb)
        conv(f"{n}.branch1x1", x, n, 0, sb)
        y = conv(f"{n}.branch7x7_1", x)
        y = conv(f"{n}.branch7x7_2", y)
        conv(f"{n}.branch7x7_3", y, n, 192, sb)
        y = conv(f"{n}.branch7x7dbl_1", x)
        for k in (2, 3, 4):
            y = conv(f"{n}.branch7x7dbl_{k}", y)
        conv(f"{n}.branch7x7dbl_5", y, n, 384, sb)
        y = pool("avg", x, f"{n}.pool", 3, 1, 1)
        conv(f"{n}.branch_pool", y, n, 576, sb)
        return n

    for n in ("Mixed_6b", "Mixed_6c", "Mixed_6d", "Mixed_6e"):
        x = mixed_c(n, x)
    n = "Mixed_7a"
    sb = T[x]["s"]
    T[n] = dict(H=8, W=8, C=1280, zp=0, s=sb)
    y = conv(f"{n}.branch3x3_1", x)
    conv(f"{n}.branch3x3_2", y, n, 0, sb)
    y = conv(f"{n}.branch7x7x3_1", x)
    y = conv(f"{n}.branch7x7x3_2", y)
    y = conv(f"{n}.branch7x7x3_3", y)
    conv(f"{n}.branch7x7x3_4", y, n, 320, sb)
    pool("max", x, n, 3, 2, 0, off=512)
    x = n

    def mixed_e(n, x):
        t = T[x]
        sb = float(np.float32(block_scale([f"{n}.branch1x1", f"{n}.branch3x3_2a", f"{n}.branch3x3dbl_3a"], x)))
        T[n] = dict(H=8, W=8, C=2048, zp=0, s=sb)
        conv(f"{n}.branch1x1", x, n, 0, sb)
        y = conv(f"{n}.branch3x3_1", x)
        conv(f"{n}.branch3x3_2a", y, n, 320, sb)
        conv(f"{n}.branch3x3_2b", y, n, 704, sb)
        y = conv(f"{n}.branch3x3dbl_1", x)
        y = conv(f"{n}.branch3x3dbl_2", y)
        conv(f"{n}.branch3x3dbl_3a", y, n, 1088, sb)
        conv(f"{n}.branch3x3dbl_3b", y, n, 1472, sb)
        y = pool("avg", x, f"{n}.pool", 3, 1, 1)
        conv(f"{n}.branch_pool", y, n, 1856, sb)
        return n

    x = mixed_e("Mixed_7b", x)
    x = mixed_e("Mixed_7c", x)
    assert len(layers) == 94
    gap = pool("avg", x, "gap", 8, 1, 0)
    g = gen.rng(seed + 99)
    fc = dict(zp_A=T[gap]["zp"], s_A=T[gap]["s"], W=gen.rand_q(g, (1000, 2048), "s8", -127, 127),
              s_W=g.uniform(0.002, 0.02, size=1000).astype(np.float32),
              bias=g.integers(-4096, 4097, size=1000).astype(np.int32))
    image = gen.rng(seed + 98).standard_normal((batch, 299, 299, 3)).astype(np.float32)
    return dict(layers=layers, ops=ops, tensors=T, fc=fc, image=image, img_scale=img_scale, img_zp=img_zp,
                batch=batch, out="gap")


def shard_inception(m, lo: int, hi: int):
    return dict(m, image=m["image"][lo:hi], batch=hi - lo)


class GpuInceptionV3:
    """The Inception-v3 forward on the library's ops (branch convs write into channel slices of
    the concat buffers), captured as one CUDA graph."""

    def __init__(self, m, dev):
        import torch

        from paper_2006_10226_b200 import qnn
        self.torch, self.qnn, self.m = torch, qnn, m
        B = m["batch"]
        T = m["tensors"]
        self.buf = {name: torch.empty((B, t["H"], t["W"], t["C"]), dtype=torch.uint8, device=dev)
                    for name, t in T.items() if name != "image"}
        self.ops = {}
        for name, L in m["layers"].items():
            c = L["c"]
            dst = [o for o in m["ops"] if o.get("name") == name][0]["dst"]
            ocs = T[dst]["C"] if dst != name else 0
            self.ops[name] = qnn.PackedConv2d(B, c.H, c.W, c.C, torch.from_numpy(L["W"]).to(dev),
                                              torch.from_numpy(L["bias"]).to(dev), L["zp_A"], 0, L["s_A"], L["s_W"],
                                              L["out"], c.stride, c.pad, (1, 1), 1, out_cstride=ocs)
        self.image_d = torch.from_numpy(m["image"]).to(dev)
        self.buf["image"] = torch.empty(self.image_d.shape, dtype=torch.uint8, device=dev)
        fc = m["fc"]
        self.fc = qnn.PackedDense(B, torch.from_numpy(fc["W"]).to(dev), torch.from_numpy(fc["bias"]).to(dev),
                                  fc["zp_A"], 0, fc["s_A"], fc["s_W"], None)
        self.fc_out = torch.empty((B, 1000), dtype=torch.int32, device=dev)
        self.logit_scale = (np.float32(fc["s_A"]) * fc["s_W"].astype(np.float32)).astype(np.float32)
        self.logits = torch.empty(self.fc_out.shape, dtype=torch.float32, device=dev)
        self.graph = None

    def step(self):
        q, m = self.qnn, self.m
        q.qnn_quantize(self.image_d, [m["img_scale"]], [m["img_zp"]], "u8", out=self.buf["image"])
        for o in m["ops"]:
            if o["kind"] == "conv":
                self.ops[o["name"]](self.buf[o["src"]], out=self.buf[o["dst"]], out_channel_offset=o["off"])
            else:
                p = o["pad"]
                q.qnn_pool2d(self.buf[o["src"]], o["kind"], o["R"], o["R"], (o["stride"],) * 2, (p, p, p, p),
                             out=self.buf[o["dst"]], out_channel_offset=o["off"])
        g = self.buf[m["out"]]
        self.fc(g.view(g.shape[0], -1), out=self.fc_out)
        q.qnn_dequantize(self.fc_out, self.logit_scale, [0], axis=-1, out=self.logits)

    def capture(self):
        torch = self.torch
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        self.qnn.launch_counter_reset()
        with torch.cuda.graph(self.graph):
            self.step()
        self.launches_per_step = self.qnn.launch_counter()
        torch.cuda.synchronize()

    def replay(self):
        self.graph.replay()

    def total_macs(self):
        return sum(L["c"].macs(self.m["batch"]) for L in self.m["layers"].values()) + self.m["batch"] * 2048 * 1000


def oracle_inception_forward(m, n_img: int = 1, with_buffers: bool = False):
    """The oracle on the Inception-v3 forward of inception_v3_full_model (NHWC between ops)."""
    import oracle as orc
    nchw = lambda t: np.ascontiguousarray(t.transpose(0, 3, 1, 2))
    nhwc = lambda t: np.ascontiguousarray(t.transpose(0, 2, 3, 1))
    T = m["tensors"]
    buf = {"image": orc.quantize(m["image"][:n_img], [m["img_scale"]], [m["img_zp"]], "u8")}
    for name, t in T.items():
        if name != "image":
            buf[name] = np.zeros((n_img, t["H"], t["W"], t["C"]), np.uint8)
    for o in m["ops"]:
        x = buf[o["src"]]
        if o["kind"] == "conv":
            L = m["layers"][o["name"]]
            c = L["c"]
            y = nhwc(orc.qnn_conv2d(nchw(x), nchw(L["W"]), L["zp_A"], 0, L["s_A"], L["s_W"], L["bias"], L["out"],
                                    c.stride, c.pad))
        else:
            p = o["pad"]
            y = nhwc(orc.pool2d(nchw(x), o["kind"], o["R"], o["R"], (o["stride"],) * 2, (p, p, p, p)))
        buf[o["dst"]][..., o["off"]:o["off"] + y.shape[-1]] = y
    g = buf[m["out"]]
    fc = m["fc"]
    acc = orc.qnn_dense(g.reshape(g.shape[0], -1), fc["W"], fc["zp_A"], 0, fc["s_A"], fc["s_W"], fc["bias"], None)
    scale = (np.float32(fc["s_A"]) * fc["s_W"]).astype(np.float32)
    if with_buffers:
        return orc.dequantize(acc, scale, [0], axis=-1), acc, buf
    return orc.dequantize(acc, scale, [0], axis=-1)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no_samples"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- oracle (CPU) arm
def oracle_forward(model, n_img: int = 1):
    """The oracle, as it stands, on n_img images of the same workload (NCHW)."""
    import oracle as orc
    outs = {}
    img = model["image"][:n_img]
    q_img = orc.quantize(img, [model["img_scale"]], [model["img_zp"]], "u8")
    for sp in model["specs"]:
        if sp.name == "conv1":
            x = q_img
        elif sp.src:
            x = outs[sp.src]
        else:
            x = model["fresh"][sp.name][:n_img]
        W = model["weights"][sp.name]
        y = orc.qnn_conv2d(np.ascontiguousarray(x.transpose(0, 3, 1, 2)), np.ascontiguousarray(W.transpose(0, 3, 1, 2)),
                           sp.zp_A, sp.zp_W, sp.s_A, sp.s_W, model["biases"][sp.name], sp.out, sp.stride, sp.pad)
        outs[sp.name] = np.ascontiguousarray(y.transpose(0, 2, 3, 1))
    fc = model["fc"]
    acc = orc.qnn_dense(fc["A"][:n_img], fc["W"], fc["zp_A"], 0, fc["s_A"], fc["s_W"], fc["bias"], None)
    scale = (np.float32(fc["s_A"]) * fc["s_W"]).astype(np.float32)
    return orc.dequantize(acc, scale, [0], axis=-1), outs


def oracle_full_forward(m, n_img: int = 1):
    """The oracle on the full forward of resnet50_full_model (NHWC in/out at each op)."""
    import oracle as orc
    nchw = lambda t: np.ascontiguousarray(t.transpose(0, 3, 1, 2))
    nhwc = lambda t: np.ascontiguousarray(t.transpose(0, 2, 3, 1))

    def conv(name, x):
        L = m["layers"][name]
        c = L["c"]
        y = orc.qnn_conv2d(nchw(x), nchw(L["W"]), L["zp_A"], 0, L["s_A"], L["s_W"], L["bias"], L["out"], c.stride,
                           c.pad)
        return nhwc(y)

    x = orc.quantize(m["image"][:n_img], [m["img_scale"]], [m["img_zp"]], "u8")
    x = conv("conv1", x)
    x = nhwc(orc.pool2d(nchw(x), "max", 3, 3, (2, 2), (1, 1, 1, 1)))
    for b in m["blocks"]:
        n = b["name"]
        y2 = conv(n + ".conv2", conv(n + ".conv1", x))
        sc = conv(n + ".downsample", x) if b["down"] else x
        (zc, sc3), (zs, ss), (zy, sy) = b["c3"], b["sc"], b["y"]
        if b["fused"]:
            L = m["layers"][n + ".conv3"]
            c = L["c"]
            x = nhwc(orc.qnn_conv2d_add(nchw(y2), nchw(L["W"]), L["zp_A"], 0, L["s_A"], L["s_W"], L["bias"],
                                        nchw(sc), ss, zs, L["out"], c.stride, c.pad))
        else:
            x = orc.add(conv(n + ".conv3", y2), sc3, zc, sc, ss, zs, sy, zy, "u8", "upward", relu=True)
    x = nhwc(orc.pool2d(nchw(x), "avg", 7, 7))
    fc = m["fc"]
    acc = orc.qnn_dense(x.reshape(x.shape[0], -1), fc["W"], fc["zp_A"], 0, fc["s_A"], fc["s_W"], fc["bias"], None)
    scale = (np.float32(fc["s_A"]) * fc["s_W"]).astype(np.float32)
    return orc.dequantize(acc, scale, [0], axis=-1)


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_single_thread_rates():
    """the oracle's single-thread rate on C1 (the 3x3 16->16 conv at 8x8, batch 1)
    and C4-512 (qnn.dense 512^3), int64 MAC/s, each repeated for about a second."""
    import oracle as orc
    from workloads import gen
    n0 = orc.num_threads()
    orc.set_num_threads(1)
    try:
        c = gen.conv_case(101, 1, 16, 8, 8, 16, 3, 3, (1, 1), (1, 1, 1, 1), relu=False, zp_A=128, zp_out=128)
        macs1 = 64 * 16 * 144
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < 1.0:
            orc.qnn_conv2d(c.nchw(), c.oihw(), c.zp_A, c.zp_W, c.s_A, c.s_W, c.bias, c.out_params(), c.stride, c.pad)
            reps += 1
        dt1 = (time.perf_counter() - t0) / reps
        d = gen.dense_case(3512, 512, 512, 512)
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < 1.0 or reps == 0:
            orc.qnn_dense(d.A, d.W, d.zp_A, d.zp_W, d.s_A, d.s_W, d.bias, d.out_params())
            reps += 1
        dt4 = (time.perf_counter() - t0) / reps
    finally:
        orc.set_num_threads(n0)
    return {"C1_us": round(dt1 * 1e6, 1), "C1_gmacs": round(macs1 / dt1 / 1e9, 3),
            "C4_512_ms": round(dt4 * 1e3, 2), "C4_512_gmacs": round(512 ** 3 / dt4 / 1e9, 3), "threads": 1}


def cpu_baseline(model, n_img: int = 1):
    import oracle as orc
    t0 = time.perf_counter()
    oracle_forward(model, n_img)
    dt = time.perf_counter() - t0
    macs = sum(sp.N * sp.P * sp.Q * sp.K * sp.R * sp.S * sp.C for sp in model["specs"]) / max(1, model["specs"][0].N)
    out = {"value": n_img / dt, "unit": "images/s", "cores": orc.num_threads(), "kind": "oracle",
           "sample": f"{n_img} image(s) through the full stack (quantize, 53 conv, fc, dequantize), {dt:.1f} s",
           "gmacs": round(n_img * macs / dt / 1e9, 2), "cpu": _cpu_model(),
           "affinity_cores": len(os.sched_getaffinity(0))}
    try:
        out["single_thread"] = oracle_single_thread_rates()
    except Exception as e:    # a timing extra: never fail the bench line for it
        out["single_thread"] = {"error": str(e)[:200]}
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return
    model = resnet50_model(1)
    if args.warmup > 0:
        oracle_forward(model, 1)          # one untimed pass (bounded: the oracle is slow)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle_forward(model, 1)
        times.append(time.perf_counter() - t0)
    import oracle as orc
    tot = sum(times)
    value = args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "per_step_sample": "1 image (bounded CPU sample of the 256-image step)",
                       "global_batch": 1, "parallelism": "cpu oracle, rank 0 only"},
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": orc.num_threads(), "kind": "oracle",
                             "sample": f"{args.steps} steps x 1 image through the full stack"},
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- main
def _spawn_ranks(args) -> int:
    """--gpus N > 1 without torchrun: launch the N ranks ourselves (one process per GPU)."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _peaks():
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    mma = {}
    try:
        mma = json.load(open(os.path.join(ROOT, "profiles", "mma_peak.json")))
    except (OSError, ValueError):
        pass
    return peaks, mma


def _layer_roofline_us(macs: float, nbytes: float, tc_tops: float, hbm_gbs: float) -> float:
    """min-time of one launch on the measured roofline: max(ops / TC peak, bytes / HBM peak)."""
    return max(2.0 * macs / (tc_tops * 1e12), nbytes / (hbm_gbs * 1e9)) * 1e6


def _time_replays(torch, replay, steps, world, dist, dev):
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        replay()
    t1.record()
    torch.cuda.synchronize()
    from paper_2006_10226_b200.sharding import max_over_ranks
    return max_over_ranks(t0.elapsed_time(t1), dist if world > 1 else None, dev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--global-batch", type=int, default=256,
                    help="configs[4]: images per step over ALL GPUs (strong scaling: 256 / N per GPU)")
    ap.add_argument("--impl", default="qnn", choices=["qnn", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--breakdown-steps", type=int, default=5)
    ap.add_argument("--no-full-network", dest="full_network", action="store_false",
                    help="skip the full-forward (glue ops) measurement")
    ap.add_argument("--no-weak", dest="weak", action="store_false", help="skip the weak-scaling figure (N > 1)")
    ap.add_argument("--no-inception", dest="inception", action="store_false",
                    help="skip the Inception-v3 full-forward measurement")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "contract: at least 3 warm-up steps"

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2006_10226_b200.sharding import max_over_ranks, shard_range
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    G = args.global_batch
    lo, hi = shard_range(G, rank, world)
    gmodel = resnet50_model(G)
    model = shard_model(gmodel, lo, hi)
    batch = hi - lo
    net = GpuResNet50(model, dev)
    net.capture()
    for _ in range(args.warmup):
        net.replay()
    torch.cuda.synchronize()

    # ---------------- timed region: K graph replays, inputs resident in HBM (strong scaling)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    ms = _time_replays(torch, net.replay, args.steps, world, dist, dev)
    clk = clocks.stop()
    ms_per_step = ms / args.steps
    value = G * args.steps / (ms / 1000.0)

    # ---------------- e2e: host f32 image in -> logits out on the host, same metric, through the
    # C-ABI host-buffer entry points: every step, qnn_quantize_host copies the step's f32 images
    # from pinned host memory (copy engine, copy stream) into a device staging buffer and
    # quantizes them on the compute stream; the graph (53 conv + fc) ends in qnn_dequantize_host,
    # which writes the f32 logits straight into pinned host memory.  Two staging buffers: step
    # k+1's copy overlaps step k's graph.  The timed region starts before the first copy and ends
    # after the last logits reached the host.
    from paper_2006_10226_b200 import qnn_quantize_host
    host_in = torch.from_numpy(model["image"]).pin_memory()
    host_out = torch.empty(net.logits.shape, dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 50))
    net.capture_e2e(host_out)
    staging = (torch.empty_like(net.image_d), torch.empty_like(net.image_d))
    cstream, copy_s = torch.cuda.current_stream(), torch.cuda.Stream()
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    img_scale, img_zp = [model["img_scale"]], [model["img_zp"]]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cstream)
    copy_s.wait_event(e0)
    for k in range(e2e_steps):
        b = k & 1
        if k >= 2:
            copy_s.wait_event(consumed[b])   # step k-2's quantize is done with this staging buffer
        qnn_quantize_host(host_in, staging[b], net.q_image, img_scale, img_zp, "u8", copy_stream=copy_s,
                          stream=cstream)
        consumed[b].record(cstream)
        net.graph_e2e.replay()
    e1.record(cstream)
    torch.cuda.synchronize()
    ems = max_over_ranks(e0.elapsed_time(e1), dist if world > 1 else None, dev)
    e2e_value = G * e2e_steps / (ems / 1000.0)
    # the last step's logits, read from the host buffer, equal the device-timed graph's
    e2e_ok = bool(torch.equal(host_out, net.logits.cpu()))
    h2d = host_in.numel() * 4
    d2h = host_out.numel() * 4

    # ---------------- per-layer breakdown: each layer captured as its own CUDA graph and
    # replayed back to back, bracketed by CUDA events on the launching stream (no host gaps)
    nl = len(net.stack.specs)
    layer_graphs = []
    for sp in net.stack.specs:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            net.stack.ops[sp.name](net.stack.inputs[sp.name], out=net.stack.outs[sp.name])
        layer_graphs.append(g)
    fc_graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(fc_graph):
        net.fc(net.fc_in, out=net.fc_out)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(nl + 1)]
    layer_ms = np.zeros(nl)
    fc_ms = 0.0
    for _ in range(args.breakdown_steps):
        for i, g in enumerate(layer_graphs + [fc_graph]):
            evs[i][0].record()
            g.replay()
            evs[i][1].record()
        torch.cuda.synchronize()
        t = np.array([a.elapsed_time(b) for a, b in evs])
        layer_ms += t[:nl]
        fc_ms += t[nl]
    layer_ms /= args.breakdown_steps
    fc_ms /= args.breakdown_steps
    macs = [sp.macs() for sp in net.stack.specs]
    fcW = model["fc"]["W"]
    fc_macs = batch * fcW.shape[0] * fcW.shape[1]
    # GEMM time of a step: the 54 GEMM launches captured as ONE graph (exactly the step's
    # kernels minus quantize/dequantize), replayed back to back between two events
    gg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gg):
        net.stack.run()
        net.fc(net.fc_in, out=net.fc_out)
    for _ in range(2):
        gg.replay()
    torch.cuda.synchronize()
    reps = max(3, args.breakdown_steps)
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    for _ in range(reps):
        gg.replay()
    g1.record()
    torch.cuda.synchronize()
    gemm_ms = g0.elapsed_time(g1) / reps
    gemm_ops = 2.0 * (sum(macs) + fc_macs)
    gemm_launches = nl + 1
    peaks, mma = _peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    bf16_burst = peaks.get("bf16_tflops", 1590.0)
    bf16_sus = peaks.get("bf16_tflops_sustained", 1400.0)
    # the guide's rule: int8 peak = measured bf16 x nominal 4.5/2.25; the burst figure when the
    # timed region ran at (near) max SM clock, the sustained one when it ran throttled
    sm_mhz, sm_max = clk.get("sm_mhz"), clk.get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)
    burst = sm_mhz is None or sm_mhz >= 0.95 * sm_max
    int8_peak = 2.0 * (bf16_burst if burst else bf16_sus)
    achieved = gemm_ops / (gemm_ms / 1000.0) / 1e12
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "gemm_traffic.json")))
        if tr.get("batch") == batch:
            traffic = tr.get("bytes_per_launch")
    except (OSError, ValueError):
        pass
    step_ops = 2.0 * (net.stack.total_macs() + fc_macs)
    conv_tops = step_ops / (ms_per_step / 1000.0) / 1e12 * world
    # per-layer roofline (algorithmic bytes = input once + weights + output + 12 B/channel)
    layer_bytes = [sp.N * sp.H * sp.W * sp.C + sp.K * sp.C * sp.R * sp.S + sp.N * sp.P * sp.Q * sp.K + 12 * sp.K
                   for sp in net.stack.specs]
    roof_us = [_layer_roofline_us(m, b, int8_peak, hbm) for m, b in zip(macs, layer_bytes)]
    fc_bytes = batch * fcW.shape[1] + fcW.size + batch * fcW.shape[0] * 4 + 12 * fcW.shape[0]
    fc_roof_us = _layer_roofline_us(fc_macs, fc_bytes, int8_peak, hbm)
    roof_sum_us = sum(roof_us) + fc_roof_us
    mma_peak = None
    if mma.get("int8_macs_per_clk_per_sm") and sm_mhz:
        mma_peak = 2.0 * mma["int8_macs_per_clk_per_sm"] * mma.get("sm_count", 148) * sm_mhz * 1e6 / 1e12

    # ---------------- weak scaling (N > 1): 256 images per GPU, same recipe
    weak = None
    if world > 1 and args.weak:
        wmodel = resnet50_model(G)
        wnet = GpuResNet50(wmodel, dev)
        wnet.capture()
        for _ in range(3):
            wnet.replay()
        wsteps = max(3, min(args.steps, 50))
        wms = _time_replays(torch, wnet.replay, wsteps, world, dist, dev)
        weak = {"value": round(G * world * wsteps / (wms / 1000.0), 1), "unit": "images/s",
                "per_gpu_batch": G, "ms_per_step": round(wms / wsteps, 4), "steps": wsteps}
        del wnet

    # ---------------- full network: the same convs plus max pool, 16 residual
    # qnn.add and global average pool between them; reported alongside, not as `value`
    full = None
    if args.full_network:
        fm = shard_full_model(resnet50_full_model(G), lo, hi)
        fnet = GpuResNet50Full(fm, dev)
        fnet.capture()
        for _ in range(3):
            fnet.replay()
        torch.cuda.synchronize()
        fsteps = max(3, min(args.steps, 50))
        fms = _time_replays(torch, fnet.replay, fsteps, world, dist, dev) / fsteps
        full = {"value": round(G / (fms / 1000.0), 1), "unit": "images/s",
                "ms_per_step": round(fms, 4), "steps": fsteps, "launches_per_step": fnet.launches_per_step,
                "ops": "quantize, conv1, max pool 3x3/2, 16 x (3-4 conv, the residual qnn.add + ReLU fused into "
                       "conv3's epilogue), global avg pool, fc, dequantize"}
        del fnet

    # ---------------- Inception-v3 full forward (configs[4]'s second network), same global batch
    incep = None
    if args.inception:
        im = shard_inception(inception_v3_full_model(G), lo, hi)
        inet = GpuInceptionV3(im, dev)
        inet.capture()
        for _ in range(3):
            inet.replay()
        torch.cuda.synchronize()
        isteps = max(3, min(args.steps, 50))
        ims = _time_replays(torch, inet.replay, isteps, world, dist, dev) / isteps
        incep = {"value": round(G / (ims / 1000.0), 1), "unit": "images/s", "ms_per_step": round(ims, 4),
                 "steps": isteps, "launches_per_step": inet.launches_per_step,
                 "conv_tops": round(2.0 * inet.total_macs() * world / (ims / 1000.0) / 1e12, 1),
                 "ops": "quantize (299x299x3 f32 -> u8), 94 conv (branch outputs written into channel slices "
                        "of the concat buffers), 4 max pools, 9 branch avg pools, global avg pool, fc, dequantize"}
        del inet

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(model, 1)
    layers = [{"name": sp.name, "ms": round(float(t), 4), "tops": round(2.0 * m / (t / 1000.0) / 1e12, 1),
               "roof_us": round(r, 1), "frac_roofline": round(r / (t * 1000.0), 3)}
              for sp, t, m, r in zip(net.stack.specs, layer_ms, macs, roof_us)]
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
        "config": {"workload": WORKLOAD, "global_batch": G, "per_gpu_batch": batch,
                   "image": "224x224x3 f32 -> u8", "parallelism": f"dp{world} (batch {G} sharded {G}/{world} per GPU, "
                   "replicated weights, no data-path collective)", "weights": "s8 symmetric per-channel",
                   "activations": "u8", "rounding": "UPWARD",
                   "l2": "no flush: per-step working set (154 MB f32 input + ~1.9 GB activations at batch 256) "
                         "exceeds the 126 MB L2", "graph": "CUDA graph replay per step"},
        "conv_tops": round(conv_tops, 1), "conv_pct_int8_peak": round(100 * conv_tops / int8_peak, 2),
        "e2e": {"value": round(e2e_value, 1), "unit": "images/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "api": "C-ABI qnn_quantize_host (pinned f32 in, copy engine) + graph + qnn_dequantize_host (f32 logits "
                       "written into pinned host memory)", "logits_match_device_step": e2e_ok,
                "note": "every step: pinned f32 images H2D (copy engine, double-buffered: step k+1's copy "
                        "overlaps step k) + quantize + graph + f32 logits to pinned host memory"},
        "gpu_launches": int(net.launches_per_step * args.steps),
        "roofline": {"kernel": "tcgen05 GEMMs: qnn_gemm_i8_kernel + qnn_gemm_t_kernel (all 54 conv/fc launches "
                               "of a step)", "bound": "tensor",
                     "achieved": round(achieved, 1), "peak": round(int8_peak, 1), "unit": "TOPS",
                     "frac": round(achieved / int8_peak, 4),
                     "peak_note": ("int8 dense = 2 x measured %s bf16 (MEASURED_PEAKS.json), the guide's nominal "
                                   "4.5/2.25 ratio; %s because the timed region ran at %s MHz of %s") %
                                  ("burst" if burst else "sustained", "burst" if burst else "sustained", sm_mhz, sm_max),
                     "roofline_sum_frac": round(roof_sum_us / (gemm_ms * 1000.0), 4),
                     "roofline_sum_us": round(roof_sum_us, 1),
                     "roofline_sum_note": "sum over the 54 launches of max(ops / int8 peak, algorithmic bytes / "
                                          "measured HBM) divided by the measured GEMM time of a step (SURVEY §8d C5)",
                     "peak_mma_microbench": None if mma_peak is None else round(mma_peak, 1),
                     "frac_mma_microbench": None if mma_peak is None else round(achieved / mma_peak, 4),
                     "mma_note": "tools/micro/mma_rate.cu: tcgen05.mma kind::i8 M=128 N=256 issue rate "
                                 "(profiles/mma_peak.json) x 148 SMs x the timed region's median SM clock",
                     "traffic": traffic, "launches_per_step": gemm_launches,
                     "kernel_share_of_step": round(gemm_ms / ms_per_step, 3),
                     "ops_per_step": gemm_ops},
        "clocks": clk,
        "cpu_baseline": cpu,
        "weak_scaling": weak,
        "full_network": full,
        "inception_v3": incep,
        "layers": layers,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
