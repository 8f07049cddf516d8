import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return round(s.elapsed_time(e) * 1e3 / reps, 2)
for lg in (27, 28, 29, 30):
    x = ops.fill_synthetic("f32_unit", 1 << lg, seed=1)
    r = {"n": lg}
    for block, grid in ((256, 0), (512, 0), (1024, 0), (1024, 148), (1024, 296), (512, 296), (512, 592)):
        r[f"{block}x{grid}"] = t(lambda: ops.reduce_sum_f32(x, block=block, grid=grid))
    print(json.dumps(r), flush=True)
    del x
