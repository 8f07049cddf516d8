"""Raw pinned host -> device bandwidth on the box vs the e2e reduce path."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)
n = 1 << 30
x = ops.fill_synthetic("f32_unit", n, seed=1)
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h.copy_(x)
d = torch.empty_like(x)
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
el = (time.perf_counter() - t) / 3
print("raw H2D GB/s", round(4 * n / el / 1e9, 2))
ops.reduce_sum_f32_host(h)
t = time.perf_counter()
for _ in range(3):
    ops.reduce_sum_f32_host(h)
el = (time.perf_counter() - t) / 3
print("e2e reduce GB/s", round(4 * n / el / 1e9, 2), "Gelem/s", round(n / el / 1e9, 3))
