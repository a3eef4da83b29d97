#!/usr/bin/env python
"""the two lowerings of a u8 x u8 (TFLite-style per-tensor, zp_W != 0)
conv on tcgen05 -- direct u8 x u8 MMA vs the VNNI Legalize (weights requantized to
s8, zp_W - 128) -- timed on ResNet-50 b256 layer shapes with CUDA events (L2 not flushed: the
per-launch working set is above the 126 MB L2 for these layers).  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2006_10226_b200 import PackedConv2d  # noqa: E402
from paper_2006_10226_b200.qnn import legalize_s8_weights  # noqa: E402
from workloads import gen  # noqa: E402
from workloads.shapes import resnet50_unique  # noqa: E402


def main(batch=256, reps=20):
    rows = []
    for c in resnet50_unique():
        if c.name not in ("layer1.0.conv2", "layer2.0.conv1", "layer3.1.conv2", "layer4.1.conv2", "layer1.0.conv3"):
            continue
        g = gen.rng(11)
        A = torch.from_numpy(gen.rand_q(g, (batch, c.H, c.W, c.C), "u8")).cuda()
        Wu = torch.from_numpy(gen.rand_q(g, (c.K, c.R, c.S, c.C), "u8")).cuda()
        zpW, zpA, sA, sW = 121, 128, 0.02, [0.004]
        out = dict(scale=gen.calibrated_out_scale(c.C * c.R * c.S, (0, 255), zpA, (0, 255), zpW, sA, sW[0]),
                   zero_point=0, dtype="u8", rounding="upward", relu=True)
        Ws, zp2 = legalize_s8_weights(Wu, zpW)
        res = {"layer": c.name}
        ys = []
        for tag, w, zp in (("u8xu8", Wu, zpW), ("u8xs8_legalized", Ws, zp2)):
            op = PackedConv2d(batch, c.H, c.W, c.C, w, None, zpA, zp, sA, sW, out, c.stride, c.pad)
            y = op(A)
            for _ in range(3):
                op(A, out=y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                op(A, out=y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            res[tag + "_us"] = round(ms * 1000, 2)
            res[tag + "_tops"] = round(2.0 * c.macs(batch) / (ms / 1000) / 1e12, 1)
            ys.append(y.clone())
        res["identical"] = bool(torch.equal(ys[0], ys[1]))
        rows.append(res)
    print(json.dumps({"batch": batch, "zp_W": 121, "note": "zp_W != 0: Term 3 row sums on both lowerings",
                      "layers": rows}))


if __name__ == "__main__":
    main()
