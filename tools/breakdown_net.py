"""Per-op device time of the full forwards (ResNet-50 with glue, Inception-v3) at one batch:
each op captured as its own CUDA graph and replayed back to back between CUDA events (no L2
flush: the steady state inside a step).  Prints one JSON line per op, sorted by time.

  python tools/breakdown_net.py inception 256
  python tools/breakdown_net.py resnet50_full 256
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def time_graph(fn, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    net_name, B = sys.argv[1], int(sys.argv[2])
    dev = torch.device("cuda")
    rows = []
    if net_name == "inception":
        m = bench.inception_v3_full_model(B)
        net = bench.GpuInceptionV3(m, dev)
        net.step()
        q = net.qnn
        for o in m["ops"]:
            if o["kind"] == "conv":
                L = m["layers"][o["name"]]
                fn = (lambda o=o: net.ops[o["name"]](net.buf[o["src"]], out=net.buf[o["dst"]],
                                                     out_channel_offset=o["off"]))
                macs = L["c"].macs(B)
                name = o["name"]
            else:
                p = o["pad"]
                fn = (lambda o=o, p=p: q.qnn_pool2d(net.buf[o["src"]], o["kind"], o["R"], o["R"], (o["stride"],) * 2,
                                                    (p, p, p, p), out=net.buf[o["dst"]], out_channel_offset=o["off"]))
                macs = 0
                name = f"{o['kind']}pool {o['src']}->{o['dst']}"
            ms = time_graph(fn)
            rows.append(dict(name=name, us=round(ms * 1000, 1), tops=round(2 * macs / (ms / 1e3) / 1e12, 1)))
    else:
        m = bench.resnet50_full_model(B)
        net = bench.GpuResNet50Full(m, dev)
        net.step()
        # whole forward, then glue ops alone
        rows.append(dict(name="full forward", us=round(time_graph(net.step) * 1000, 1)))
        q = net.qnn
        rows.append(dict(name="maxpool", us=round(time_graph(lambda: q.qnn_pool2d(
            net.buf["conv1"], "max", 3, 3, (2, 2), (1, 1, 1, 1), out=net.pool)) * 1000, 1)))
        rows.append(dict(name="gap", us=round(time_graph(lambda: q.qnn_pool2d(
            net.buf[m["blocks"][-1]["name"] + ".out"], "avg", 7, 7, out=net.gap)) * 1000, 1)))
        for b in m["blocks"]:
            n = b["name"]
            sc = net.buf[n + ".downsample"] if b["down"] else (net.pool if n == "layer1.0" else None)
            if sc is None:
                prev = [x for x in m["blocks"] if x["name"] < n]
                sc = net.buf[prev[-1]["name"] + ".out"] if prev else net.pool
            scq = b["sc"]
            rows.append(dict(name=n + ".conv3+residual", us=round(time_graph(
                lambda n=n, sc=sc, scq=scq: net.ops[n + ".conv3"](net.buf[n + ".conv2"], out=net.buf[n + ".out"],
                                                                residual=(sc, scq[1], scq[0]))) * 1000, 1)))
    tot = sum(r["us"] for r in rows if r["name"] != "full forward")
    for r in sorted(rows, key=lambda r: -r["us"]):
        print(json.dumps(r))
    print(json.dumps(dict(name="SUM", us=round(tot, 1))))


if __name__ == "__main__":
    main()
