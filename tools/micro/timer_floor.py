"""Floor of tools/bench_layers.Timer: a graph with one trivial kernel, and N back-to-back copies."""
import torch
from tools.bench_layers import Timer
t = Timer()
x = torch.zeros(1, device="cuda")
print("1 tiny kernel  :", round(t.time(lambda: x.add_(1), 40) * 1e3, 2), "us")
def ten():
    for _ in range(10):
        x.add_(1)
print("10 tiny kernels:", round(t.time(ten, 40) * 1e3, 2), "us")
