"""Timing of the reference-formulation native kernels (dsl/patterns.py) at the
BASELINE sizes, for variant sweeps.  usage: WF_LIB=... python tools/patterns_probe.py"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402
from paper_2112_10034_b200.dsl import patterns  # noqa: E402

st = torch.cuda.current_stream().cuda_stream


def t(fn, it=20, r=5):
    fn()
    torch.cuda.synchronize()
    v = []
    for _ in range(r):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(it):
            fn()
        b.record()
        b.synchronize()
        v.append(a.elapsed_time(b) * 1e3 / it)
    return round(statistics.median(v), 1)


res = {"lib": Path(str(_lib.lib_path())).stem}
x = ops.fill_synthetic("f32_unit", 1 << 30, seed=1)
for grid in (148 * 8, 148 * 16, 4096):
    o = torch.empty(grid * 8, dtype=torch.float32, device="cuda")
    pw = patterns.NativePattern("warp_partials_sum_f32", "wf_warp_partials_sum_f32", "a", "out", "n")
    cfg = type("C", (), {"grid_size": grid, "block_size": 256, "warp_size": 32})()
    res[f"c2_grid{grid}_us"] = t(lambda: pw.run(cfg, {"a": x, "out": o, "n": 1 << 30}, st))
del x
x = ops.fill_synthetic("i32_full", 1 << 28, seed=0)
y = torch.empty_like(x)
pp = patterns.NativePattern("warp_prefix32_i32", "wf_warp_prefix32_i32", "a", "out")
cfg = type("C", (), {"grid_size": (1 << 28) // 256, "block_size": 256, "warp_size": 32})()
res["c3_prefix_us"] = t(lambda: pp.run(cfg, {"a": x, "out": y}, st))
res["copy_us"] = t(lambda: y.copy_(x))
print(json.dumps(res), flush=True)
