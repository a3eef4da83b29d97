#!/usr/bin/env python
"""Per-layer / per-op sweeps (BASELINE configs[1..3]) with L2 flushed between reps.

  python tools/bench_layers.py --suite resnet50 --batch 64      # configs[1]
  python tools/bench_layers.py --suite mobilenet --batch 128    # configs[2]
  python tools/bench_layers.py --suite dense                    # configs[3]
  python tools/bench_layers.py --suite requant                  # standalone requantize / quantize / dequantize
  python tools/bench_layers.py --only layer1.0.conv3 --reps 3   # one layer (for ncu)

Each line: layer, time (trimmed mean of reps, CUDA events, L2 flushed by writing a
256 MB buffer before every rep), algorithmic TOPS / GB/s, and the
fraction of the measured roofline (MEASURED_PEAKS.json: HBM copy bandwidth,
int8 = 2 x measured bf16 burst).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_10226_b200 import qnn  # noqa: E402
from workloads import gen  # noqa: E402
from workloads.shapes import mobilenet_v2_convs, resnet50_unique  # noqa: E402


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        p = {}
    return p.get("hbm_gbs", 6650.0), 2.0 * p.get("bf16_tflops", 1590.0)


class Timer:
    """Times one op as a CUDA-graph replay so host-side launch preparation (plan,
    tensor-map encoding, ctypes) never shows up as GPU time.  L2 is flushed before
    every rep by READING a 512 MB buffer (a write-based flush would leave ~126 MB
    of dirty lines whose write-back lands inside the timed op)."""

    def __init__(self, flush_mb=512, flush=True, b2b=1):
        self.flush = torch.ones(flush_mb * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
        self.sink = torch.empty((), dtype=torch.float32, device="cuda")
        # flush=False, b2b=k: the graph holds k back-to-back copies of the op and the time is per
        # copy -- the steady-state cost of a launch whose inputs / code may still be in L2 (the
        # per-launch floor of small layers: compare with the flushed single replay)
        self.do_flush, self.b2b = flush, b2b

    def time(self, fn, reps=10, warmup=3):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(self.b2b):
                fn()
        ts = []
        for _ in range(reps):
            if self.do_flush:
                torch.sum(self.flush, dim=0, out=self.sink)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) / self.b2b)
        # event timestamps tick in ~2 us steps here: a trimmed mean over many reps averages the
        # quantisation out where a median would keep it
        ts.sort()
        k = len(ts) // 10
        ts = ts[k:len(ts) - k] if len(ts) > 4 else ts
        return statistics.fmean(ts)


def conv_layer(c, batch, per_channel=True, seed=0):
    wdt, zpW = ("s8", 0) if per_channel else ("u8", 128)
    case = gen.conv_case(seed, batch, c.C, c.H, c.W, c.K, c.R, c.S, c.stride, c.pad, (1, 1), c.groups, "u8", wdt,
                         zp_W=zpW, per_channel=per_channel, relu=c.relu, act6=c.act6)
    dev = torch.device("cuda")
    op = qnn.PackedConv2d(batch, c.H, c.W, c.C, torch.from_numpy(case.W).to(dev), torch.from_numpy(case.bias).to(dev),
                          case.zp_A, case.zp_W, case.s_A, case.s_W, case.out_params(), c.stride, c.pad, (1, 1),
                          c.groups)
    x = torch.from_numpy(case.A).to(dev)
    y = torch.empty(op.out_shape(), dtype=op.out_dtype, device=dev)
    macs = c.macs(batch)
    bytes_ = x.numel() + y.numel() + case.W.size + 12 * c.K
    return (lambda: op(x, out=y)), macs, bytes_


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--suite", default="resnet50", choices=["resnet50", "mobilenet", "dense", "requant", "all"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--only", default=None)
    ap.add_argument("--reps", type=int, default=40)
    ap.add_argument("--per-tensor", action="store_true", help="u8 weights with zp_W != 0 (TFLite style)")
    ap.add_argument("--json", default=None)
    ap.add_argument("--b2b", type=int, default=0, help="no L2 flush; time K back-to-back launches per replay")
    args = ap.parse_args()
    hbm, tc = peaks()
    t = Timer(flush=args.b2b == 0, b2b=max(1, args.b2b))
    rows = []

    def report(name, ms, macs=0, bytes_=0):
        tops = 2 * macs / (ms / 1e3) / 1e12 if macs else 0.0
        gbs = bytes_ / (ms / 1e3) / 1e9
        ai = 2 * macs / bytes_ if bytes_ else 0
        roof = min(tc, ai * hbm / 1e3) if macs else hbm / 1e3
        frac = (tops / roof) if macs else gbs / hbm
        r = dict(name=name, ms=round(ms, 4), tops=round(tops, 1), gbs=round(gbs, 1), ai=round(ai, 1),
                 roof_tops=round(roof, 1), frac_roofline=round(frac, 3))
        rows.append(r)
        print(json.dumps(r), flush=True)

    suites = ["resnet50", "mobilenet", "dense", "requant"] if args.suite == "all" else [args.suite]
    for suite in suites:
        if suite == "resnet50":
            for b in ([args.batch] if args.batch else [1, 64]):
                for c in resnet50_unique():
                    if args.only and c.name != args.only:
                        continue
                    fn, macs, by = conv_layer(c, b, not args.per_tensor)
                    report(f"r50_b{b}.{c.name}", t.time(fn, args.reps), macs, by)
        elif suite == "mobilenet":
            b = args.batch or 128
            seen = set()
            for c in mobilenet_v2_convs():
                key = (c.C, c.K, c.H, c.R, c.stride, c.groups)
                if key in seen or (args.only and c.name != args.only):
                    continue
                seen.add(key)
                fn, macs, by = conv_layer(c, b, True)
                report(f"mbv2_b{b}.{c.name}{'.dw' if c.groups > 1 else ''}", t.time(fn, args.reps), macs, by)
        elif suite == "dense":
            for n in (512, 1024, 2048, 4096, 8192):
                if args.only and args.only != f"dense_{n}":
                    continue
                case = gen.dense_case(3000 + n, n, n, n)
                dev = torch.device("cuda")
                op = qnn.PackedDense(n, torch.from_numpy(case.W).to(dev), torch.from_numpy(case.bias).to(dev),
                                     case.zp_A, 0, case.s_A, case.s_W, case.out_params())
                a = torch.from_numpy(case.A).to(dev)
                y = torch.empty((n, n), dtype=torch.uint8, device=dev)
                report(f"dense_{n}", t.time(lambda: op(a, out=y), args.reps), n ** 3, 3 * n * n)
        elif suite == "requant":
            n = 256 * 56 * 56 * 256 // 4
            x32 = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda")
            y8 = torch.empty(n, dtype=torch.uint8, device="cuda")
            report("requantize_s32_to_u8", t.time(lambda: qnn.qnn_requantize(x32, [0.001], 0, 1.0, 128, "u8",
                                                                               out=y8), args.reps), 0, 5 * n)
            x8 = torch.randint(0, 255, (4 * n,), dtype=torch.uint8, device="cuda")
            z8 = torch.empty(4 * n, dtype=torch.int8, device="cuda")
            report("requantize_u8_to_s8", t.time(lambda: qnn.qnn_requantize(x8, [0.3], 128, 0.2, 0, "s8", out=z8),
                                                 args.reps), 0, 8 * n)
            xf = torch.randn(n, dtype=torch.float32, device="cuda")
            report("quantize_f32_to_u8", t.time(lambda: qnn.qnn_quantize(xf, [0.02], [128], "u8", out=y8),
                                                args.reps), 0, 5 * n)
            of = torch.empty(n, dtype=torch.float32, device="cuda")
            report("dequantize_u8_to_f32", t.time(lambda: qnn.qnn_dequantize(y8, [0.02], [128], out=of),
                                                  args.reps), 0, 5 * n)
    if args.json:
        json.dump(rows, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
