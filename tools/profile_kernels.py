"""Run each hot-path kernel at its BASELINE size (warm-up + measured launch)
for ncu captures:  ncu --set full -k regex:'reduce_kernel|scan_i32|compact|hist256' ...
Usage: python tools/profile_kernels.py [c1 c2 c3 c4 c5]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

which = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
torch.cuda.set_device(0)
reps = 2
if "c1" in which:
    x = ops.fill_synthetic("i32_full", 1 << 20, seed=0)
    for _ in range(reps):
        ops.reduce_sum_i32(x, block=256)
    del x
if "c2" in which:
    x = ops.fill_synthetic("f32_unit", 1 << 30, seed=1)
    for _ in range(reps):
        ops.reduce_sum_f32(x)
    del x
if "c3" in which or "c4" in which:
    x = ops.fill_synthetic("i32_full", 1 << 28, seed=0)
    y = torch.empty_like(x)
    if "c3" in which:
        for _ in range(reps):
            ops.scan_inclusive_i32(x, y)
    if "c4" in which:
        for _ in range(reps):
            ops.compact_gt0_i32(x, y)
    del x, y
if "c5" in which:
    u = ops.fill_synthetic("u8_uniform", 1 << 32, seed=0)
    for _ in range(reps):
        ops.histogram256_u8(u)
    del u
torch.cuda.synchronize()
print("done", which)
