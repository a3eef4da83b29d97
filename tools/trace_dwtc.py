"""CTA-0 timeline of the tensor-core depthwise kernel (instrumented build: QNN_BUILD_DEFS=-DQNN_DWTC_TRACE_BUILD)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
os.environ["QNN_DWTC_TRACE"] = str(buf.data_ptr())
from tools.bench_layers import conv_layer  # noqa
from workloads.shapes import mobilenet_v2_convs
name, batch = sys.argv[1], int(sys.argv[2])
c = [x for x in mobilenet_v2_convs() if x.name == name][0]
fn, macs, by = conv_layer(c, batch)
fn(); torch.cuda.synchronize(); buf.zero_(); fn(); torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.int64)
t0 = t[8000]
r = lambda a: np.where(a > 0, a - t0, -1)
print("producer item: start, got-empty"); print(r(t[0:24]).reshape(-1, 2))
print("mma group (it): tempty wait start/end"); print(r(t[200:280]).reshape(-1, 2))
e = r(t[1000:1000 + 4 * 64]).reshape(-1, 4)[:, :3]
print("epi tile: wait-start, tfull, done"); print(e[:48])
print("end", r(t[8001:8002]))
