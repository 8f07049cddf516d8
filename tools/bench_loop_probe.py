"""Why does bench.py's C2 step differ from tools/k2_grid3.py?  Same loop with
and without the NVML clock sampler thread."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)
x = ops.fill_synthetic("f32_unit", 1 << 30, seed=1)
def loop(block, steps=20):
    for _ in range(5): ops.reduce_sum_f32(x, block=block)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps): ops.reduce_sum_f32(x, block=block)
    t1.record(); torch.cuda.synchronize()
    return round(t0.elapsed_time(t1) * 1e3 / steps, 1)
for rnd in range(2):
    for block in (256, 1024):
        plain = loop(block)
        with bench.ClockSampler(0) as clk:
            sampled = loop(block)
        print(json.dumps({"block": block, "plain_us": plain, "with_nvml_sampler_us": sampled,
                          "samples": clk.summary()["samples"]}))
