"""C1 end to end through wf_reduce_sum_i32_host: pinned vs pageable host
input at 2^16 .. 2^24 (median of 50 synchronous calls, host clock), result
checked.  usage: [WF_LIB=...] python tools/zc_probe.py"""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
res = {"lib": Path(str(_lib.lib_path())).stem}
for lg in (16, 20, 22, 24):
    n = 1 << lg
    x = ops.fill_synthetic("i32_full", n, seed=3)
    want = int(x.to(torch.int64).sum().item())
    want = ((want + (1 << 31)) % (1 << 32)) - (1 << 31)
    pinned = torch.empty(n, dtype=torch.int32, pin_memory=True)
    pinned.copy_(x)
    page = pinned.numpy().copy()
    row = {}
    for name, h in (("pinned", pinned), ("pageable", page)):
        got = ops.reduce_sum_i32_host(h, device=dev)
        ok = got == want
        ts = []
        for _ in range(50):
            t = time.perf_counter()
            ops.reduce_sum_i32_host(h, device=dev)
            ts.append(time.perf_counter() - t)
        m = statistics.median(ts)
        row[name] = {"us": round(m * 1e6, 1), "gelem_s": round(n / m / 1e9, 2), "ok": ok}
    res[f"2^{lg}"] = row
print(json.dumps(res), flush=True)
