"""K3 / K4 per launch, back to back (20 launches between two events), plain
vs WF_FLAG_INPUT_STABLE, rounds interleaved, at the BASELINE size and the
8-GPU shard size.  usage: WF_LIB=... python tools/tmem_pdl_probe.py [log2n ...]"""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

torch.cuda.set_device(0)


def one(fn, it=20):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / it


for lg in [int(v) for v in sys.argv[1:]] or [25, 28]:
    x = ops.fill_synthetic("i32_full", 1 << lg, seed=3)
    y = torch.empty_like(x)
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    variants = {"scan": lambda: ops.scan_inclusive_i32(x, y),
                "scan_pdl": lambda: ops.scan_inclusive_i32(x, y, input_stable=True),
                "compact": lambda: ops.compact_gt0_i32(x, y, cnt),
                "compact_pdl": lambda: ops.compact_gt0_i32(x, y, cnt, input_stable=True)}
    for fn in variants.values():
        one(fn, 3)
    times = {k: [] for k in variants}
    for _ in range(7):
        for k, fn in variants.items():
            times[k].append(one(fn))
    res = {"lib": Path(str(_lib.lib_path())).stem, "log2n": lg}
    res.update({k + "_us": round(statistics.median(v), 1) for k, v in times.items()})
    print(json.dumps(res), flush=True)
    del x, y
