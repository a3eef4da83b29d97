"""Quick parity probe of the pixel-major kernel's CTA-pair mode (QNN_PAIR=1; run under a timeout)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from gpu_helpers import gpu_conv, oracle_conv, gpu_dense, oracle_dense
from workloads import gen
ok = True
cases = [(2, 64, 12, 12, 96, 3, (2, 2), (1, 1, 1, 1)), (1, 128, 9, 9, 128, 3, (1, 1), (1, 1, 1, 1)),
         (2, 256, 9, 7, 256, 3, (2, 2), (1, 1, 1, 1)), (1, 512, 7, 7, 512, 3, (1, 1), (1, 1, 1, 1)),
         (2, 96, 10, 10, 48, 1, (2, 2), (0, 0, 0, 0)), (2, 256, 11, 13, 512, 1, (2, 2), (0, 0, 0, 0))]
for i, (N, C, H, W, K, R, st, pad) in enumerate(cases):
    for mode in ("upward", "tonearest"):
        c = gen.conv_case(1300 + i, N, C, H, W, K, R, R, st, pad, (1, 1), 1, "u8", "s8", rounding=mode)
        _, _, y = gpu_conv(c)
        torch.cuda.synchronize()
        r = np.array_equal(y.cpu().numpy(), oracle_conv(c))
        print((N, C, H, W, K, R, st, mode), r, flush=True)
        ok &= r
d = gen.dense_case(77, 300, 512, 1024, out_dtype="s32")
_, _, y = gpu_dense(d)
r = np.array_equal(y.cpu().numpy(), oracle_dense(d)); print("dense s32", r); ok &= r
print("OK" if ok else "MISMATCH")
