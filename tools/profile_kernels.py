"""Run each hot-path kernel at its BASELINE size (warm-up + measured launch)
for ncu captures:  ncu --set full -k regex:'reduce_kernel|scan_i32|compact|hist256' ...
Usage: python tools/profile_kernels.py [c1 c2 c3 c4 c5]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

which = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5", "ref"]
torch.cuda.set_device(0)
reps = 2
if "c1" in which:
    x = ops.fill_synthetic("i32_full", 1 << 20, seed=0)
    for _ in range(reps):
        ops.reduce_sum_i32(x, block=256)
    del x
if "c2" in which:
    x = ops.fill_synthetic("f32_unit", 1 << 30, seed=1)
    for _ in range(reps):
        ops.reduce_sum_f32(x)
    del x
if "c3" in which or "c4" in which:
    x = ops.fill_synthetic("i32_full", 1 << 28, seed=0)
    y = torch.empty_like(x)
    if "c3" in which:
        for _ in range(reps):
            ops.scan_inclusive_i32(x, y)
    if "c4" in which:
        for _ in range(reps):
            ops.compact_gt0_i32(x, y)
    del x, y
if "ref" in which:  # the reference's own formulations (dsl/patterns.py native kernels)
    from paper_2112_10034_b200.dsl import patterns
    pw = patterns.NativePattern("warp_partials_sum_f32", "wf_warp_partials_sum_f32", "a", "out", "n")
    pp = patterns.NativePattern("warp_prefix32_i32", "wf_warp_prefix32_i32", "a", "out")
    x = ops.fill_synthetic("f32_unit", 1 << 30, seed=1)
    o = torch.empty(148 * 8 * 8, dtype=torch.float32, device="cuda")
    cfg = type("C", (), {"grid_size": 148 * 8, "block_size": 256, "warp_size": 32})()
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(reps):
        pw.run(cfg, {"a": x, "out": o, "n": 1 << 30}, st)
    del x, o
    x = ops.fill_synthetic("i32_full", 1 << 28, seed=0)
    y = torch.empty_like(x)
    cfg = type("C", (), {"grid_size": (1 << 28) // 256, "block_size": 256, "warp_size": 32})()
    for _ in range(reps):
        pp.run(cfg, {"a": x, "out": y}, st)
    del x, y
if "c5" in which:
    u = ops.fill_synthetic("u8_uniform", 1 << 32, seed=0)
    for _ in range(reps):
        ops.histogram256_u8(u)
    del u
torch.cuda.synchronize()
print("done", which)
