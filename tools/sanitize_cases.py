"""Small cases through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck) runs: BASELINE config 1, the channel-major pointwise GEMM (+ fused residual), the
staged-row 3x3 GEMM, the smem-built stem, im2col with border classes, zp_W != 0 (Term-3 sums),
dense, TMA depthwise, the tensor-core depthwise, requantize / quantize / dequantize, add, pool.
Each output is also compared with the oracle (exit status 1 on a mismatch)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as orc  # noqa: E402
from gpu_helpers import gpu_conv, oracle_conv  # noqa: E402
from paper_2006_10226_b200 import qnn  # noqa: E402
from workloads import gen  # noqa: E402

bad = 0
cases = [
    ("config1", gen.conv_case(101, 1, 16, 8, 8, 16, 3, 3, (1, 1), (1, 1, 1, 1), zp_A=128)),
    ("pointwise_t", gen.conv_case(111, 2, 64, 6, 7, 256, 1, 1)),
    ("rows3x3", gen.conv_case(112, 1, 64, 10, 9, 64, 3, 3, (1, 1), (1, 1, 1, 1))),
    ("stem", gen.conv_case(113, 1, 3, 32, 32, 64, 7, 7, (2, 2), (3, 3, 3, 3))),
    ("im2col_s2", gen.conv_case(114, 2, 128, 9, 9, 128, 3, 3, (2, 2), (1, 1, 1, 1))),
    ("zpw", gen.conv_case(115, 2, 64, 7, 7, 64, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), 1, "u8", "u8", zp_W=121,
                          per_channel=False)),
    ("dw_tma", gen.conv_case(116, 2, 32, 9, 8, 32, 3, 3, (1, 1), (1, 1, 1, 1), (1, 1), 32)),
    ("dw_tc", gen.conv_case(117, 1, 32, 11, 11, 32, 5, 5, (1, 1), (2, 2, 2, 2), (1, 1), 32)),
]
for name, c in cases:
    _, _, y = gpu_conv(c)
    if not np.array_equal(y.cpu().numpy(), oracle_conv(c)):
        print("MISMATCH", name)
        bad += 1
d = gen.dense_case(7, 64, 384, 256)
op = qnn.PackedDense(64, torch.from_numpy(d.W).cuda(), torch.from_numpy(d.bias).cuda(), d.zp_A, d.zp_W, d.s_A, d.s_W,
                     d.out_params())
if not np.array_equal(op(torch.from_numpy(d.A).cuda()).cpu().numpy(),
                      orc.qnn_dense(d.A, d.W, d.zp_A, d.zp_W, d.s_A, d.s_W, d.bias, d.out_params())):
    print("MISMATCH dense")
    bad += 1
x = np.random.default_rng(1).integers(-2**31, 2**31, size=10007, dtype=np.int64).astype(np.int32)
if not np.array_equal(qnn.qnn_requantize(torch.from_numpy(x).cuda(), [0.013], 0, 97.0, 128, "u8").cpu().numpy(),
                      orc.requantize(x, [0.013], 0, 97.0, 128, "u8")):
    print("MISMATCH requantize")
    bad += 1
f = np.random.default_rng(2).standard_normal(4099).astype(np.float32)
q = qnn.qnn_quantize(torch.from_numpy(f).cuda(), [0.02], [128], "u8")
if not np.array_equal(q.cpu().numpy(), orc.quantize(f, [0.02], [128], "u8")):
    print("MISMATCH quantize")
    bad += 1
dq = qnn.qnn_dequantize(q, [0.02], [128]).cpu().numpy()
if not np.array_equal(dq, orc.dequantize(q.cpu().numpy(), [0.02], [128])):
    print("MISMATCH dequantize")
    bad += 1
a = torch.from_numpy(gen.rand_q(gen.rng(3), (2, 6, 6, 32), "u8")).cuda()
b = torch.from_numpy(gen.rand_q(gen.rng(4), (2, 6, 6, 32), "u8")).cuda()
s = qnn.qnn_add(a, 0.1, 3, b, 0.2, 5, 0.25, 0, "u8", "upward", relu=True)
if not np.array_equal(s.cpu().numpy(), orc.add(a.cpu().numpy(), 0.1, 3, b.cpu().numpy(), 0.2, 5, 0.25, 0, "u8",
                                                 "upward", relu=True)):
    print("MISMATCH add")
    bad += 1
p = qnn.qnn_pool2d(a, "max", 3, 3, (2, 2), (1, 1, 1, 1))
pw = orc.pool2d(np.ascontiguousarray(a.cpu().numpy().transpose(0, 3, 1, 2)), "max", 3, 3, (2, 2), (1, 1, 1, 1))
if not np.array_equal(p.cpu().numpy(), pw.transpose(0, 2, 3, 1)):
    print("MISMATCH pool")
    bad += 1
torch.cuda.synchronize()
print("sanitize cases done, mismatches:", bad)
sys.exit(1 if bad else 0)
