python - <<'PY'
import torch, sys, statistics
sys.path.insert(0, '.')
from paper_2112_10034_b200 import ops
from oracle import numpy_oracle as no, synthetic
x = ops.fill_synthetic("f32_unit", 1 << 30, seed=1)
import os
for mode in ("0", "1"):
    os.environ["WF_RED_TMA"] = mode
    for _ in range(3): ops.reduce_sum_f32(x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); ops.reduce_sum_f32(x); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    v = float(ops.reduce_sum_f32(x).item())
    print(os.environ.get("WF_LIB", "default"), "tma", mode, "us", round(statistics.median(ts), 1), "GB/s", round(4 * (1 << 30) / statistics.median(ts) / 1e3, 1), "val", v)
n = (1 << 22) + 77
a = synthetic.generate("f32_unit", n, seed=3)
os.environ["WF_RED_TMA"] = "1"
g = float(ops.reduce_sum_f32(torch.from_numpy(a).cuda()).item())
print("small ok", abs(g - no.reduce_sum_f32_exact(a)) <= no.f32_tolerance(n, no.abs_sum(a)), g, no.reduce_sum_f32_exact(a))
PY
