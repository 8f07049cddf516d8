"""Quick CUDA-event timing of the hot-path kernels at BASELINE sizes (for
iterating on kernel variants; bench.py is the contract).
Usage: python tools/bench_kernels.py [c1 c2 c3 c4 c5] [--reps R]"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
which = args or ["c1", "c2", "c3", "c4", "c5"]
reps = 20
torch.cuda.set_device(0)


def t(fn, n_bytes, label, flush=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush:
            flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = statistics.median(ts)
    print(json.dumps({"kernel": label, "us_median": round(ms * 1e3, 2),
                      "us_min": round(min(ts) * 1e3, 2), "gbs": round(n_bytes / ms / 1e6, 1)}))


if "c1" in which:
    x = ops.fill_synthetic("i32_full", 1 << 20)
    fb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    t(lambda: ops.reduce_sum_i32(x), 4 << 20, "c1 flushed", flush=lambda: fb.fill_(1))
    t(lambda: ops.reduce_sum_i32(x), 4 << 20, "c1 warm-L2")
    del x, fb
if "c2" in which:
    x = ops.fill_synthetic("f32_unit", 1 << 30)
    t(lambda: ops.reduce_sum_f32(x), 4 << 30, "c2")
    del x
if "c3" in which or "c4" in which:
    x = ops.fill_synthetic("i32_full", 1 << 28)
    y = torch.empty_like(x)
    if "c3" in which:
        t(lambda: ops.scan_inclusive_i32(x, y), 8 << 28, "c3")
        ref = torch.cumsum(x.to(torch.int64), 0).remainder_(1 << 32)
        ok = torch.equal(ref, y.to(torch.int64).remainder_(1 << 32))
        print(json.dumps({"kernel": "c3", "correct": bool(ok)}))
        del ref
    if "c4" in which:
        t(lambda: ops.compact_gt0_i32(x, y), 6 << 28, "c4")
        _, cnt = ops.compact_gt0_i32(x, y)
        want = torch.masked_select(x, x > 0)
        m = int(cnt.item())
        print(json.dumps({"kernel": "c4", "correct": m == want.numel() and torch.equal(y[:m], want)}))
        del want
    del x, y
if "c5" in which:
    u = ops.fill_synthetic("u8_uniform", 1 << 32)
    t(lambda: ops.histogram256_u8(u), 1 << 32, "c5")
if "ref" in which:
    # library reference points on the same box: torch copy (read+write) and
    # torch.cumsum on int32 (CUB DeviceScan), both over 2^28 int32
    x = ops.fill_synthetic("i32_full", 1 << 28)
    y = torch.empty_like(x)
    t(lambda: y.copy_(x), 8 << 28, "ref torch copy 1 GiB")
    t(lambda: torch.cumsum(x, 0, out=y), 8 << 28, "ref torch.cumsum i32 (CUB)")
    t(lambda: torch.masked_select(x, x > 0), 6 << 28, "ref torch.masked_select x>0")
    del x, y
