"""Per-tile phase timestamps of the TMEM-parked scan/compaction kernel (build a
variant with -DWF_TM_TRACE=1 and point WF_LIB at it):
  0 claimed+TMA issued, 1 aggregator start, 2 parked (aggregate published),
  5 look-back warp picked it up, 3 prefix known, 4 finished,
  6 look-back polls, 7 SM id.
usage: WF_LIB=build/variants/lib_trace.so python tools/trace_tmem.py [log2n] [permille...]"""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

W = 8
torch.cuda.set_device(0)
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
sels = [int(v) for v in sys.argv[2:] if v.isdigit()] or [500]
n = 1 << log2n
x = torch.empty(n, dtype=torch.int32, device="cuda")
y = torch.empty_like(x)
nt = (n + 8191) // 8192
raw = ctypes.CDLL(str(_lib.lib_path()))


def pc(a):
    return [round(float(np.percentile(a, q)), 2) for q in (10, 50, 90, 99)]


sweep = "--lookback" not in sys.argv
sys.argv = [v for v in sys.argv if v != "--lookback"]
jobs = [("scan", None)] + [("compact", s) for s in sels]
for op, sel in jobs:
    if sel is None:
        ops.fill_synthetic("i32_full", n, out=x)
        run = lambda: ops.scan_inclusive_i32(x, y)  # noqa: E731
    else:
        ops.fill_synthetic("i32_select", n, param=sel, out=x)
        run = lambda: ops.compact_gt0_i32(x, y)  # noqa: E731
    tr = torch.zeros(nt * W, dtype=torch.int64, device="cuda")
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    us_plain = e0.elapsed_time(e1) * 100
    if not hasattr(raw, "wf_debug_set_trace_tm"):  # untraced variant: timing only
        print(json.dumps({"op": op, "sel_permille": sel, "n": n,
                          "lib": Path(str(_lib.lib_path())).stem,
                          "us_untraced": round(us_plain, 1)}), flush=True)
        continue
    raw.wf_debug_set_trace_tm(ctypes.c_void_p(tr.data_ptr()))
    run()
    torch.cuda.synchronize()
    raw.wf_debug_set_trace_tm(ctypes.c_void_p(0))
    a = tr.cpu().numpy().reshape(-1, W)
    t = a[:, :7].astype(np.float64)
    t -= t[:, 0].min()
    t /= 1e3
    mid = slice(nt // 4, 3 * nt // 4)
    tm = t[mid]
    span = t[:, 4].max()
    m = span / 2
    latest_park = np.maximum.accumulate(t[:, 2])
    latest_pref = np.maximum.accumulate(t[:, 3])
    res = {"op": op, "sel_permille": sel, "n": n, "lib": Path(str(_lib.lib_path())).stem,
           "us_untraced": round(us_plain, 1), "span_us": round(float(span), 1),
           "tiles_per_us": round(nt / float(span), 1),
           "land_wait_us(1-0)": pc(tm[:, 1] - tm[:, 0]),
           "aggregate_us(2-1)": pc(tm[:, 2] - tm[:, 1]),
           "lb_pickup_us(5-2)": pc(tm[:, 5] - tm[:, 2]),
           "lookback_us(3-5)": pc(tm[:, 3] - tm[:, 5]),
           "finish_us(4-3)": pc(tm[:, 4] - tm[:, 3]),
           "prefix_after_latest_pred_park_us": pc((t[:, 3] - latest_park)[mid]),
           "prefix_after_pred_prefix_us": pc((t[1:, 3] - latest_pref[:-1])[nt // 4:3 * nt // 4]),
           "polls": pc(a[mid, 6].astype(np.float64)),
           "at_mid": {"loading": int(((t[:, 0] <= m) & (t[:, 1] > m)).sum()),
                      "parked_wait_lb": int(((t[:, 2] <= m) & (t[:, 5] > m)).sum()),
                      "in_lookback": int(((t[:, 5] <= m) & (t[:, 3] > m)).sum()),
                      "wait_finish": int(((t[:, 3] <= m) & (t[:, 4] > m)).sum())}}
    # fill / drain: when the pipeline's fronts reach their ends, relative to
    # the first claim (all in us)
    res["fronts_us"] = {"first_land": round(float(t[:, 1].min()), 2),
                        "first_finish": round(float(t[:, 4].min()), 2),
                        "last_claim": round(float(t[:, 0].max()), 2),
                        "last_land": round(float(t[:, 1].max()), 2),
                        "last_park": round(float(t[:, 2].max()), 2),
                        "last_prefix": round(float(t[:, 3].max()), 2),
                        "end": round(float(t[:, 4].max()), 2)}
    # how far behind the claim front is the prefix front, in tiles, at mid-run
    res["at_mid"]["claimed"] = int((t[:, 0] <= m).sum())
    res["at_mid"]["prefix_known"] = int((t[:, 3] <= m).sum())
    res["at_mid"]["finished"] = int((t[:, 4] <= m).sum())
    if sweep:  # sweeper build: 5 = finisher has the item, 6 = finisher local work done
        for k in ("lb_pickup_us(5-2)", "lookback_us(3-5)", "polls"):
            res.pop(k, None)
        res["park_to_prefix_us(3-2)"] = pc(tm[:, 3] - tm[:, 2])
        res["park_to_fin_start_us(5-2)"] = pc(tm[:, 5] - tm[:, 2])
        res["fin_local_us(6-5)"] = pc(tm[:, 6] - tm[:, 5])
        res["prefix_minus_local_done_us(3-6)"] = pc(tm[:, 3] - tm[:, 6])
        res["fin_end_after_ready_us"] = pc(tm[:, 4] - np.maximum(tm[:, 3], tm[:, 6]))
        sm = a[:, 7]
        gaps = []
        for s_id in np.unique(sm):
            st = np.sort(t[sm == s_id, 5])
            gaps.append(np.diff(st))
        g = np.concatenate(gaps)
        res["fin_start_gap_per_sm_us"] = pc(g[g.size // 4: 3 * g.size // 4] if g.size > 8 else g)
    print(json.dumps(res), flush=True)
