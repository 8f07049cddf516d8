"""Steady-state check of one library (WF_LIB): per-launch time and result of
20 back-to-back scan / compaction launches on one workspace, against torch
(cumsum / masked_select).  usage: WF_LIB=... python tools/ab_check.py [log2n]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 28)
x = ops.fill_synthetic("i32_full", n)
want_scan = torch.cumsum(x.to(torch.int64), 0).to(torch.int32)  # wraps like int32 after the cast
want_c = torch.masked_select(x, x > 0)
y = torch.empty_like(x)
for op in ("scan", "compact"):
    times, bad = [], 0
    for i in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if op == "scan":
            ops.scan_inclusive_i32(x, y)
        else:
            _, c = ops.compact_gt0_i32(x, y)
        e.record()
        torch.cuda.synchronize()
        times.append(round(s.elapsed_time(e) * 1e3, 1))
        if op == "scan":
            bad += int(not torch.equal(y, want_scan))
        else:
            m = int(c.item())
            bad += int(m != want_c.numel() or not torch.equal(y[:m], want_c))
    print(json.dumps({"lib": Path(str(_lib.lib_path())).stem, "op": op, "n": n, "bad": bad,
                      "us": times}), flush=True)
