"""Run one conv layer through the channel-major GEMM with QNN_GEMM_TRACE (instrumented build:
QNN_LIB=.../libqnn_instr.so) and print CTA 0's per-tile timeline (profiling aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
os.environ["QNN_GEMM_TRACE"] = str(buf.data_ptr())
from tools.bench_layers import conv_layer  # noqa: E402
from workloads.shapes import resnet50_unique  # noqa: E402

name, batch = sys.argv[1], int(sys.argv[2])
c = [x for x in resnet50_unique() if x.name == name][0]
fn, macs, by = conv_layer(c, batch)
fn(); torch.cuda.synchronize(); buf.zero_(); fn(); torch.cuda.synchronize()
t = buf.cpu().numpy()[:448].reshape(7, 64).astype(np.int64)
t0 = t[t > 0].min()
names = ["prod_issue", "build_start", "build_done", "mma_start", "mma_commit", "epi_wake", "epi_store"]
print(name, batch, "tiles traced", int((t[5] > 0).sum()))
print("tile " + " ".join(f"{n:>11s}" for n in names))
for i in range(0, 24):
    print(f"{i:4d} " + " ".join(f"{(v - t0) if v > 0 else -1:11d}" for v in t[:, i]))
for k, n in enumerate(names):
    v = t[k][t[k] > 0]
    if v.size > 3:
        print(f"{n:12s} median period {np.median(np.diff(v)):8.0f}")
