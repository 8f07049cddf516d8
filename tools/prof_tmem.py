"""Per-role cycle accounting of the TMEM scan/compaction kernel (variant built
with -DWF_TM_PROF=1): where the finisher, the aggregator and the producer of
each CTA spend their cycles, per item, averaged over CTAs.
usage: WF_LIB=build/variants/lib_prof.so python tools/prof_tmem.py [log2n] [permille...]"""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
sels = [int(v) for v in sys.argv[2:]] or [0, 500]
n = 1 << log2n
x = torch.empty(n, dtype=torch.int32, device="cuda")
y = torch.empty_like(x)
raw = ctypes.CDLL(str(_lib.lib_path()))
jobs = [("scan", None)] + [("compact", s) for s in sels]
for op, sel in jobs:
    if sel is None:
        ops.fill_synthetic("i32_full", n, out=x)
        run = lambda: ops.scan_inclusive_i32(x, y)  # noqa: E731
    else:
        ops.fill_synthetic("i32_select", n, param=sel, out=x)
        run = lambda: ops.compact_gt0_i32(x, y)  # noqa: E731
    for _ in range(5):
        run()
    prof = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    raw.wf_debug_set_prof_tm(ctypes.c_void_p(prof.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    raw.wf_debug_set_prof_tm(ctypes.c_void_p(0))
    a = prof.cpu().numpy().reshape(148, 16).astype(np.float64)
    a = a[a[:, 5] > 0]
    per = lambda k, items: round(float((a[:, k] / np.maximum(a[:, items], 1)).mean()), 1)  # noqa: E731
    print(json.dumps({
        "op": op, "sel": sel, "n": n, "us": round(e0.elapsed_time(e1) * 1e3, 1),
        "items_per_cta": round(float(a[:, 5].mean()), 1),
        "finisher_cycles_per_item": {"wait_parked": per(0, 5), "tmem_read_free": per(1, 5),
                                     "local": per(2, 5), "wait_prefix": per(3, 5),
                                     "store": per(4, 5)},
        "aggregator0_cycles_per_item": {"wait_full": per(6, 9), "wait_slot": per(7, 9),
                                        "work": per(8, 9)},
        "producer_cycles_per_item": {"wait_empty": per(10, 12), "issue": per(11, 12)},
    }), flush=True)
