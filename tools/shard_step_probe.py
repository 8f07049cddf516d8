"""Per-rank step of every sharded BASELINE config at the shard sizes of
1/2/4/8 GPUs (strong scaling of the fixed BASELINE job), measured on one B200
with the world-1 protocol of the fused kernels (the exchange's flag / fence /
poll protocol runs; NVLink latency does not), steps back to back as
programmatic dependent launches exactly as bench.py times them.  The
predicted speed-up at N GPUs is t(1) / t(N) (the NVLink round trip of the
exchange, ~1-2 us, comes on top at N > 1).  Variants interleaved by round.
usage: python tools/shard_step_probe.py"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops, p2p  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
boxes = p2p.Mailboxes.local(1, dev, cap=256)
pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)
kboxes = p2p.Mailboxes.local(1, dev)
pr = p2p.PeerReducer(kboxes[0], 0, 1)


def one(fn, it=20):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / it


rows = {}
for N in (1, 2, 4, 8):
    f = ops.fill_synthetic("f32_unit", (1 << 30) // N, seed=1)
    x = ops.fill_synthetic("i32_full", (1 << 28) // N, seed=0)
    y = torch.empty_like(x)
    u = ops.fill_synthetic("u8_uniform", (1 << 32) // N, seed=0)
    torch.cuda.synchronize()
    if N == 1:  # the single-GPU paths bench.py times at N = 1
        v = {"C2": lambda: ops.reduce_sum_f32(f, input_stable=True),
             "C3": lambda: ops.scan_inclusive_i32(x, y, input_stable=True),
             "C4": lambda: ops.compact_gt0_i32(x, y, input_stable=True),
             "C5": lambda: ops.histogram256_u8(u, input_stable=True)}
    else:  # the fused per-rank kernels bench.py runs at N > 1
        def c3():
            c = pc.reduce_exscan_i32(x, input_stable=True)[:1]
            ops.scan_inclusive_i32(x, y, carry=c, input_stable=True)
        v = {"C2": lambda: pr.reduce_sum_f32(f, input_stable=True),
             "C3": c3,
             "C4": lambda: pc.compact_gt0_i32(x, y, input_stable=True),
             "C5": lambda: pc.histogram256_u8(u, input_stable=True)}
    for fn in v.values():
        one(fn, 3)
    t = {k: [] for k in v}
    for _ in range(5):
        for k, fn in v.items():
            t[k].append(one(fn))
    rows[N] = {k: statistics.median(vals) for k, vals in t.items()}
    torch.cuda.synchronize()
    del f, x, y, u
out = {}
for cfg in ("C2", "C3", "C4", "C5"):
    t1 = rows[1][cfg]
    out[cfg] = {f"N{N}": {"step_us": round(rows[N][cfg], 1),
                          "speedup": round(t1 / rows[N][cfg], 2),
                          "efficiency": round(t1 / rows[N][cfg] / N, 3)} for N in rows}
print(json.dumps(out), flush=True)
assert not pc.failed()
boxes[0].close()
kboxes[0].close()
