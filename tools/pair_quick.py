"""Quick parity probe of the channel-major kernel's CTA-pair mode (run under a timeout)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from gpu_helpers import gpu_conv, oracle_conv
from workloads import gen
ok = True
for (N, C, H, W, K) in [(2, 64, 9, 7, 256), (1, 128, 10, 10, 256), (2, 256, 13, 11, 512), (1, 64, 5, 5, 256),
                        (2, 1024, 7, 7, 256), (1, 512, 7, 9, 1024)]:
    c = gen.conv_case(900 + K + C, N, C, H, W, K, 1, 1)
    _, _, y = gpu_conv(c)
    torch.cuda.synchronize()
    r = np.array_equal(y.cpu().numpy(), oracle_conv(c))
    print((N, C, H, W, K), "M", N * H * W, r, flush=True)
    ok &= r
print("OK" if ok else "MISMATCH")
