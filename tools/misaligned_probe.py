"""Scan / compaction throughput on 4-byte (not 16-byte) aligned views at
2^28: the register-tile single-pass kernel of wf_scan.cu."""
import json, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)
n = 1 << 28
x = ops.fill_synthetic("i32_full", n + 4, seed=1)
y = torch.empty_like(x)
def t(fn):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    return round(statistics.median(ts), 1)
for off, yoff in ((0, 0), (1, 1), (1, 2)):
    xv, yv = x[off:off + n], y[yoff:yoff + n]
    print(json.dumps({"offset_elems": off, "out_offset": yoff, "scan_us": t(lambda: ops.scan_inclusive_i32(xv, yv)),
                      "compact_us": t(lambda: ops.compact_gt0_i32(xv, yv))}))
