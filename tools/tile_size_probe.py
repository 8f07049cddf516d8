"""Fixed vs per-tile cost of K3 / K4: back-to-back step time over sizes
2^13 .. 2^28 (plain and dependent launches), and the least-squares line
t = a + b * tiles over the shard sizes (2^22 .. 2^25) — `a` is what a launch
costs regardless of size (prologue, ramp, drain), `b` the steady tile rate.
usage: python tools/tile_size_probe.py [sel_permille]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

torch.cuda.set_device(0)
sel = int(sys.argv[1]) if len(sys.argv) > 1 else 500
TILE = 8192


def graph_of(fn, it):
    """`it` back-to-back calls captured in one CUDA graph: the host's per-call
    cost (Python, ctypes) cannot hide the small sizes' device time."""
    fn()  # workspace allocated outside the capture
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(it):
                fn()
    torch.cuda.synchronize()
    return g


def one(g, it):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / it


xs_full = ops.fill_synthetic("i32_full", 1 << 28, seed=0)
xs_sel = ops.fill_synthetic("i32_select", 1 << 28, param=sel, seed=0)
y = torch.empty_like(xs_full)
res = {}
for lg in (13, 16, 19, 20, 21, 22, 23, 24, 25, 26, 28):
    torch.cuda.empty_cache()
    n = 1 << lg
    x3, x4 = xs_full[:n], xs_sel[:n]
    v = {"scan": lambda: ops.scan_inclusive_i32(x3, y),
         "scan_dep": lambda: ops.scan_inclusive_i32(x3, y, input_stable=True),
         "compact": lambda: ops.compact_gt0_i32(x4, y),
         "compact_dep": lambda: ops.compact_gt0_i32(x4, y, input_stable=True)}
    it = max(10, min(200, (1 << 30) // (n * 4)))
    gs = {k: graph_of(fn, it) for k, fn in v.items()}
    for g in gs.values():
        one(g, it)
    t = {k: [] for k in v}
    for _ in range(5):
        for k, g in gs.items():
            t[k].append(one(g, it))
    del gs
    res[lg] = {k: round(float(np.median(s)), 2) for k, s in t.items()}
    print(json.dumps({"log2n": lg, "tiles": n // TILE, **res[lg]}), flush=True)

fit = {}
for k in ("scan", "scan_dep", "compact", "compact_dep"):
    lgs = [22, 23, 24, 25]
    tiles = np.array([(1 << g) / TILE for g in lgs])
    us = np.array([res[g][k] for g in lgs])
    b, a = np.polyfit(tiles, us, 1)
    fit[k] = {"fixed_us": round(float(a), 2), "us_per_tile": round(float(b), 5),
              "tiles_per_us": round(float(1 / b), 1)}
print(json.dumps({"sel_permille": sel, "fit_2^22..2^25": fit}), flush=True)
