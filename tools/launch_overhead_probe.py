"""Where the host time of one `runtime.launch` of a small DSL kernel goes
(GPU box).  Prints per-launch wall time and a cProfile top list."""
import cProfile
import pstats
import time

import torch

from paper_2112_10034_b200 import benchmarks as bm
from paper_2112_10034_b200.config import LaunchConfig
from paper_2112_10034_b200.dsl import hybrid_transform
from paper_2112_10034_b200.memory import DeviceMemory
from paper_2112_10034_b200.runtime import launch

mem = DeviceMemory(0)
args = bm._mode_setup("veccopy", 1, 32, mem)
cfg = LaunchConfig(grid_size=1, block_size=32)
prog = hybrid_transform(bm._kernel(bm.MODE_SOURCES["veccopy"]), cfg, mode="hier")
for _ in range(50):
    launch(prog, cfg, mem, args)
N = 3000
t = time.perf_counter()
for _ in range(N):
    launch(prog, cfg, mem, args)
print(f"runtime.launch: {(time.perf_counter() - t) / N * 1e6:.1f} us")
s = torch.cuda.current_stream()
t = time.perf_counter()
for _ in range(N):
    s.synchronize()
print(f"idle stream.synchronize: {(time.perf_counter() - t) / N * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    launch(prog, cfg, mem, args)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
