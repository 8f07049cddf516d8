import json, sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)
def t(fn, reps=20):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps
for lg in (27, 30):
    x = ops.fill_synthetic("f32_unit", 1 << lg, seed=1)
    cfgs = ((256, 0), (512, 0), (1024, 0), (1024, 148))
    res = {c: [] for c in cfgs}
    for c in cfgs:
        for _ in range(3): ops.reduce_sum_f32(x, block=c[0], grid=c[1])
    for rnd in range(6):
        for c in (cfgs if rnd % 2 == 0 else cfgs[::-1]):
            res[c].append(t(lambda: ops.reduce_sum_f32(x, block=c[0], grid=c[1])))
    print(json.dumps({"n": lg, **{f"{b}x{g}": round(statistics.median(v), 2) for (b, g), v in res.items()}}), flush=True)
    del x
