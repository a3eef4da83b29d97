"""Probe HBM read/write mixes with torch ops (context for the elementwise rooflines)."""
import torch
from tools.bench_layers import Timer
t = Timer()
n = 256 * 56 * 56 * 256 // 4
f = torch.empty(n, dtype=torch.float32, device="cuda")
u = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
u2 = torch.empty_like(u)
f2 = torch.randn(n, device="cuda")
def rep(name, ms, by):
    print(f"{name:28s} {ms*1e3:8.1f} us  {by/ms/1e6:8.1f} GB/s")
rep("fill f32 (write only)", t.time(lambda: f.fill_(1.0), 20), 4 * n)
rep("copy u8->u8", t.time(lambda: u2.copy_(u), 20), 2 * n)
rep("copy f32->f32", t.time(lambda: f.copy_(f2), 20), 8 * n)
rep("u8->f32 convert", t.time(lambda: f.copy_(u), 20), 5 * n)
rep("f32->u8 convert", t.time(lambda: u2.copy_(f2), 20), 5 * n)
rep("sum f32 (read only)", t.time(lambda: f2.sum(), 20), 4 * n)
