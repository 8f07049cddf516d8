import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)
x = ops.fill_synthetic("f32_unit", 1 << 30, seed=1)
block = int(sys.argv[1])
res = []
for rnd in range(8):
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(10): ops.reduce_sum_f32(x, block=block)
    t1.record(); torch.cuda.synchronize()
    res.append(round(t0.elapsed_time(t1) * 1e3 / 10, 1))
print(block, res)
