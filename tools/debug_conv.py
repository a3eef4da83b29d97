import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from gpu_helpers import gpu_conv, oracle_conv
from test_gpu_conv import config1_case
from workloads import gen
for pad in (1, 0):
    for relu in (False, True):
        c = config1_case(pad, relu, "upward")
        _, _, y = gpu_conv(c)
        g = y.cpu().numpy(); w = oracle_conv(c)
        print("pad", pad, "relu", relu, "mismatch", (g != w).sum(), "of", g.size, "got", g.reshape(-1)[:8], "want", w.reshape(-1)[:8])
c = gen.conv_case(5, 1, 16, 8, 8, 16, 3, 3, (1, 1), (1, 1, 1, 1), out_dtype="s32")
_, _, y = gpu_conv(c); g = y.cpu().numpy(); w = oracle_conv(c)
print("s32 pad1 mismatch", (g != w).sum(), g.reshape(-1)[:4], w.reshape(-1)[:4])
c = gen.conv_case(6, 2, 64, 17, 17, 96, 1, 1, (1, 1), (0, 0, 0, 0), out_dtype="u8", relu=False)
_, _, y = gpu_conv(c); g = y.cpu().numpy(); w = oracle_conv(c)
print("1x1 u8 mismatch", (g != w).sum(), g.reshape(-1)[:8], w.reshape(-1)[:8])
# slow path: m >= 2^-1 (rsh <= 32) and tiny m (rsh > 52)
for s_out in (1e-6, 1e-4, 50.0):
    c = gen.conv_case(7, 1, 16, 8, 8, 32, 3, 3, (1, 1), (1, 1, 1, 1), relu=False)
    c.s_out = s_out
    _, _, y = gpu_conv(c); g = y.cpu().numpy(); w = oracle_conv(c)
    print("s_out", s_out, "mismatch", (g != w).sum(), g.reshape(-1)[:8], w.reshape(-1)[:8])
