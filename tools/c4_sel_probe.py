"""K4 per launch at 2^28 over selectivities (i32_select, permille), plain
launches back to back, rounds interleaved.  usage: WF_LIB=... python
tools/c4_sel_probe.py"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

torch.cuda.set_device(0)
n = 1 << 28
perms = (0, 1, 10, 30, 100, 500, 1000)
xs = {p: ops.fill_synthetic("i32_select", n, seed=0, param=p) for p in perms}
out = torch.empty(n, dtype=torch.int32, device="cuda")
cnt = torch.empty(1, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()


def one(x, it=10):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it):
        ops.compact_gt0_i32(x, out, cnt)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / it


times = {p: [] for p in perms}
for p in perms:
    one(xs[p], 2)
for _ in range(5):
    for p in perms:
        times[p].append(one(xs[p]))
ok = {}
for p in perms:
    o, c = ops.compact_gt0_i32(xs[p], out, cnt)
    want = torch.masked_select(xs[p], xs[p] > 0)
    ok[p] = int(c.item()) == want.numel() and torch.equal(o[:want.numel()], want)
print(json.dumps({"lib": Path(str(_lib.lib_path())).stem,
                  "us": {f"{p / 10:g}%": round(statistics.median(v), 1) for p, v in times.items()},
                  "ok": all(ok.values())}), flush=True)
