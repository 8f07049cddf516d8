import sys, statistics, json
sys.path.insert(0, '.')
import torch
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)
x1 = ops.fill_synthetic("i32_full", 1 << 20, seed=0)
tiny = ops.fill_synthetic("i32_full", 4, seed=0)
fb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fb.fill_(1)
res = {}
for name, flush in (("write_flush", lambda: fb.fill_(1)), ("read_flush", lambda: fb.sum(dtype=torch.int64)),
                    ("none", lambda: None)):
    for lab, x in (("2^20", x1), ("4elem", tiny)):
        ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(30)]
        for a, b in ev:
            flush()
            a.record()
            ops.reduce_sum_i32(x, block=256)
            b.record()
        torch.cuda.synchronize()
        res[f"{name}/{lab}"] = round(statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev[5:]), 2)
print(json.dumps(res))
# cold inputs without a flush kernel: 64 different 4 MiB inputs (256 MiB >
# L2) reduced back to back, two events around the whole rotation
bufs = [ops.fill_synthetic("i32_full", 1 << 20, seed=s) for s in range(64)]
outs = torch.empty(64, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
for rnd in range(3):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for k in range(64):
        ops.reduce_sum_i32(bufs[k], outs[k:k + 1], block=256)
    b.record()
    b.synchronize()
    res[f"rotating_cold_b2b_round{rnd}"] = round(a.elapsed_time(b) * 1e3 / 64, 2)
print(json.dumps(res))
