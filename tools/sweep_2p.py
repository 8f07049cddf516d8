# ROUND-1 RECORD: drove the runtime switch WF_SCAN_2P, which round 2 removed from the
# product library; the two-pass kernels now build only as variants
# (python tools/build_variants.py tp="-DWF_SCAN_IMPL=3"), selected with WF_LIB.
"""Two-pass (L2-streamed) vs single-pass scan/compaction: correctness at ragged
sizes and CUDA-event timing at 2^28, over chunk sizes (WF_2P_CHUNK_TILES) and
library variants (WF_LIB).  Usage: python tools/sweep_2p.py [chunks...]"""
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

torch.cuda.set_device(0)
chunks = [int(a) for a in sys.argv[1:]] or [512]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return round(statistics.median(ts), 2), round(min(ts), 2)


def check(n, seed=0):
    x = ops.fill_synthetic("i32_full", n, seed=seed)
    y = torch.empty_like(x)
    ops.scan_inclusive_i32(x, y)
    ref = torch.cumsum(x.to(torch.int64), 0)
    ok_scan = torch.equal((ref & 0xFFFFFFFF), y.to(torch.int64) & 0xFFFFFFFF)
    out = torch.empty_like(x)
    _, cnt = ops.compact_gt0_i32(x, out)
    m = int(cnt.item())
    want = x[x > 0]
    ok_c = m == want.numel() and torch.equal(out[:m], want)
    return bool(ok_scan), bool(ok_c)


os.environ["WF_SCAN_2P"] = "1"
lib = os.environ.get("WF_LIB", "default")
for c in chunks:
    os.environ["WF_2P_CHUNK_TILES"] = str(c)
    oks = [check(n, s) for s, n in enumerate(((1 << 22) + 5, (1 << 24) + 8191, 3 << 24))]
    n = 1 << 28
    x = ops.fill_synthetic("i32_full", n)
    y = torch.empty_like(x)
    res = {"lib": Path(lib).stem, "chunk_tiles": c, "correct": oks}
    for mode in ("1", "0"):
        os.environ["WF_SCAN_2P"] = mode
        res[f"scan_us_2p{mode}"] = timeit(lambda: ops.scan_inclusive_i32(x, y))
        res[f"compact_us_2p{mode}"] = timeit(lambda: ops.compact_gt0_i32(x, y))
    os.environ["WF_SCAN_2P"] = "1"
    res["full_correct"] = check(n, 7)
    print(json.dumps(res), flush=True)
    del x, y
    torch.cuda.empty_cache()
