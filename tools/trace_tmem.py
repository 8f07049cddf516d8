"""Per-tile phase timestamps of the TMEM-parked scan/compaction kernel (build
with -DWF_TM_TRACE=1, WF_LIB=...): 0 claimed+TMA issued, 1 aggregator start,
2 parked (aggregate handed to look-back), 3 prefix known, 4 finished."""
import ctypes
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

torch.cuda.set_device(0)
n = 1 << 28
x = ops.fill_synthetic("i32_full", n)
y = torch.empty_like(x)
nt = n // 8192
raw = ctypes.CDLL(str(_lib.lib_path()))
for op in ("scan", "compact"):
    run = (lambda: ops.scan_inclusive_i32(x, y)) if op == "scan" else (lambda: ops.compact_gt0_i32(x, y))
    tr = torch.zeros(nt * 5, dtype=torch.int64, device="cuda")
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    raw.wf_debug_set_trace_tm(ctypes.c_void_p(tr.data_ptr()))
    run()
    torch.cuda.synchronize()
    raw.wf_debug_set_trace_tm(ctypes.c_void_p(0))
    t = tr.cpu().numpy().reshape(-1, 5).astype(np.float64)
    t -= t[:, 0].min()
    t /= 1e3
    mid = slice(nt // 4, 3 * nt // 4)
    pc = lambda a: [round(float(np.percentile(a[mid], q)), 2) for q in (10, 50, 90, 99)]  # noqa: E731
    span = t[:, 4].max()
    m = span / 2
    res = {"op": op, "lib": Path(str(_lib.lib_path())).stem, "span_us": round(float(span), 1),
           "land_wait_us(1-0)": pc(t[:, 1] - t[:, 0]), "aggregate_us(2-1)": pc(t[:, 2] - t[:, 1]),
           "lookback_us(3-2)": pc(t[:, 3] - t[:, 2]), "finish_us(4-3)": pc(t[:, 4] - t[:, 3]),
           "prefix_after_latest_pred_park_us": pc(t[:, 3] - np.maximum.accumulate(t[:, 2])),
           "at_mid": {"loading": int(((t[:, 0] <= m) & (t[:, 1] > m)).sum()),
                      "parked_wait_prefix": int(((t[:, 2] <= m) & (t[:, 3] > m)).sum()),
                      "wait_finish": int(((t[:, 3] <= m) & (t[:, 4] > m)).sum())}}
    print(json.dumps(res), flush=True)
