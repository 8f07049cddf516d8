"""Per-tile phase timestamps of the scan kernel (build with -DWF_TRACE=1):
0 = ticket taken, 1 = aggregate known, 2 = prefix resolved, 3 = stores issued."""
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
ntiles = n // int(os.environ.get('WF_TRACE_TILE', '4096'))
tr = torch.zeros(ntiles * 4, dtype=torch.int64, device="cuda")
lib = _lib.load()
raw = ctypes.CDLL(str(_lib.lib_path()))
op = os.environ.get("WF_TRACE_OP", "scan")
run = (lambda: ops.scan_inclusive_i32(x, y)) if op == "scan" else (lambda: ops.compact_gt0_i32(x, y))
for _ in range(3):
    run()
raw.wf_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
run()
torch.cuda.synchronize()
raw.wf_debug_set_trace(ctypes.c_void_p(0))
t = tr.cpu().numpy().reshape(-1, 4).astype(np.float64)
t -= t[:, 0].min()
t /= 1e3  # us
load = t[:, 1] - t[:, 0]
wait = t[:, 2] - t[:, 1]
store = t[:, 3] - t[:, 2]
life = t[:, 3] - t[:, 0]
res = {"op": op, "lib": os.environ.get("WF_LIB", ""), "kernel_span_us": float(t[:, 3].max()),
       "load_compute_us": [float(np.percentile(load, q)) for q in (10, 50, 90, 99)],
       "lookback_wait_us": [float(np.percentile(wait, q)) for q in (10, 50, 90, 99)],
       "store_us": [float(np.percentile(store, q)) for q in (10, 50, 90, 99)],
       "lifetime_us": [float(np.percentile(life, q)) for q in (10, 50, 90, 99)]}
# frontier: prefix-resolved time vs tile index
order = np.argsort(t[:, 2])
res["resolved_tiles_per_us_mid"] = float(ntiles / 2 / (t[order[3 * ntiles // 4], 2] - t[order[ntiles // 4], 2]))
starts = np.sort(t[:, 0])
res["start_rate_tiles_per_us_mid"] = float(ntiles / 2 / (starts[3 * ntiles // 4] - starts[ntiles // 4]))
# lag between ticket order and resolution: how many tiles were waiting at mid-run
mid = t[:, 3].max() / 2
res["tiles_in_flight_mid"] = int(((t[:, 0] <= mid) & (t[:, 3] > mid)).sum())
res["tiles_waiting_lookback_mid"] = int(((t[:, 1] <= mid) & (t[:, 2] > mid)).sum())
res["tiles_loading_mid"] = int(((t[:, 0] <= mid) & (t[:, 1] > mid)).sum())
print(json.dumps(res))
np.save(f"gpurun_out/{op}_trace_{Path(os.environ.get('WF_LIB', 'x')).stem}.npy", t.astype(np.float32))
