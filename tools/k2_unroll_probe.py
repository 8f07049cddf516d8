"""K2 at 2^30 with 512-thread CTAs, back-to-back launches (the bench's
timed-region shape): median of 7 rounds of 20.  WF_LIB selects a variant."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

x = ops.fill_synthetic("f32_unit", 1 << 30)
out = torch.empty(1, dtype=torch.float32, device="cuda")
for _ in range(30):
    ops.reduce_sum_f32(x, out, block=512)
torch.cuda.synchronize()
v = []
for _ in range(7):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        ops.reduce_sum_f32(x, out, block=512)
    b.record()
    b.synchronize()
    v.append(a.elapsed_time(b) * 1e3 / 20)
print(f"{statistics.median(v):.1f} us  ({4 * 2**30 / statistics.median(v) / 1e3:.0f} GB/s)")
