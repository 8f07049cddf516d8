"""K2 at the 8-GPU shard size (2^27): fixed cost vs grid, and the floor."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)

def t(fn, reps=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return round(s.elapsed_time(e) * 1e3 / reps, 2)

x = ops.fill_synthetic("f32_unit", 1 << 27, seed=1)
small = x[:4096]
print(json.dumps({"floor_4096": t(lambda: ops.reduce_sum_f32(small))}))
for block, grid in ((256, 0), (256, 148), (256, 296), (256, 592), (256, 1480), (512, 296), (512, 444), (1024, 148), (1024, 296), (128, 1480)):
    print(json.dumps({"block": block, "grid": grid, "us": t(lambda: ops.reduce_sum_f32(x, block=block, grid=grid))}))
