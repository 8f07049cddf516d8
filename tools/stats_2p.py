# ROUND-1 RECORD: drove the runtime switch WF_SCAN_2P, which round 2 removed from the
# product library; the two-pass kernels now build only as variants
# (python tools/build_variants.py tp="-DWF_SCAN_IMPL=3"), selected with WF_LIB.
"""Where does the two-pass kernel's time go?  Needs a -DWF_2P_STATS=1 build
(WF_LIB=...).  Prints per-launch wait statistics at 2^28 for scan and compaction."""
import ctypes
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

torch.cuda.set_device(0)
raw = ctypes.CDLL(str(_lib.lib_path()))
buf = (ctypes.c_ulonglong * 8)()
n = 1 << 28
x = ops.fill_synthetic("i32_full", n)
y = torch.empty_like(x)
for name, fn in (("scan", lambda: ops.scan_inclusive_i32(x, y)),
                 ("compact", lambda: ops.compact_gt0_i32(x, y))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    raw.wf_debug_2p_stats(buf, 1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    raw.wf_debug_2p_stats(buf, 1)
    v = list(buf)
    print(json.dumps({"op": name, "lib": Path(str(_lib.lib_path())).stem,
                      "chunk": os.environ.get("WF_2P_CHUNK_TILES"), "us": round(s.elapsed_time(e) * 1e3, 1),
                      "p2_wait_frac_of_cta_time": round(v[0] / max(v[6], 1), 3),
                      "p2_waited_items": v[3], "p1_items": v[4], "p2_items": v[5],
                      "p2_wait_us_per_waiting_item": round(v[0] / max(v[3], 1) / 1e3, 2),
                      "chunk_lookback_us_total": round(v[1] / 1e3, 1),
                      "finisher_us_total": round(v[2] / 1e3, 1),
                      "lead_bounded_prefetches": v[7],
                      "cta_life_us_avg": round(v[6] / 1e3 / 592, 1)}), flush=True)
