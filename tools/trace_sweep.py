"""Sweeper iteration trace (variant built with -DWF_TM_TRACE=1): iteration
durations and ready-run lengths for scan / compaction at 2^28.
usage: WF_LIB=build/variants/lib_trace.so python tools/trace_sweep.py"""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

n = 1 << 28
x = ops.fill_synthetic("i32_full", n)
y = torch.empty_like(x)
raw = ctypes.CDLL(str(_lib.lib_path()))
cap = 1 << 16
for op in ("scan", "compact"):
    run = (lambda: ops.scan_inclusive_i32(x, y)) if op == "scan" else (lambda: ops.compact_gt0_i32(x, y))
    for _ in range(5):
        run()
    tr = torch.zeros(2 * cap, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    raw.wf_debug_set_trace_sweep(ctypes.c_void_p(tr.data_ptr()), ctypes.c_uint32(cap))
    run()
    torch.cuda.synchronize()
    raw.wf_debug_set_trace_sweep(ctypes.c_void_p(0), ctypes.c_uint32(0))
    a = tr.cpu().numpy().reshape(-1, 2)
    a = a[a[:, 0] != 0]
    t = (a[:, 0] - a[0, 0]) / 1e3
    ready = (a[:, 1] >> 32).astype(np.int64)
    dt = np.diff(t)
    mid = slice(len(dt) // 4, 3 * len(dt) // 4)
    pc = lambda v: [round(float(np.percentile(v, q)), 3) for q in (10, 50, 90, 99)]  # noqa: E731
    print(json.dumps({"lib": Path(str(_lib.lib_path())).stem, "op": op, "iterations": len(a),
                      "span_us": round(float(t[-1]), 1), "iter_us": pc(dt[mid]),
                      "ready": pc(ready[1:][mid]), "zero_ready_frac": round(float((ready == 0).mean()), 3),
                      "tiles_per_us_mid": round(float(ready[1:][mid].sum() / dt[mid].sum()), 1)}), flush=True)
