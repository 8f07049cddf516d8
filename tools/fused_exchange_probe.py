"""Cost of the exchange step, fused vs separate kernel, on one GPU (world-1
mailboxes: the fence / flag / poll protocol runs, NVLink latency does not).
Shard sizes = the 8-GPU shards of the BASELINE configs.  Back-to-back
launches between two CUDA events, median of 7 rounds of 50."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops, p2p  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
boxes = p2p.Mailboxes.local(1, dev, cap=256)
kboxes = p2p.Mailboxes.local(1, dev)
pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)
pr = p2p.PeerReducer(kboxes[0], 0, 1)


def timed(fn, iters=50, rounds=7):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / iters)
    return statistics.median(ts)


f = ops.fill_synthetic("f32_unit", 1 << 27, seed=1)
x = ops.fill_synthetic("i32_full", 1 << 25, seed=2)
u = ops.fill_synthetic("u8_uniform", 1 << 29, seed=3)
out = torch.empty_like(x)
cnt = torch.empty(1, dtype=torch.int64, device=dev)
rows = [
    ("C2 2^27 f32: K2 + fold kernel", lambda: ops.fold(ops.reduce_sum_f32(f, block=512))),
    ("C2 2^27 f32: K2 with exchange fused", lambda: pr.reduce_sum_f32(f, block=512)),
    ("C3 pass 1 2^25: K1 + exchange kernel", lambda: pc.exscan_u32(ops.reduce_sum_i32(x))),
    ("C3 pass 1 2^25: K1 with exchange fused", lambda: pc.reduce_exscan_i32(x)),
    ("C4 2^25: compaction + exchange kernel", lambda: pc.exscan_u64(ops.compact_gt0_i32(x, out, cnt)[1])),
    ("C4 2^25: compaction with exchange fused", lambda: pc.compact_gt0_i32(x, out)),
    ("C5 2^29 u8: histogram + exchange kernel", lambda: pc.allreduce_u64(ops.histogram256_u8(u))),
    ("C5 2^29 u8: histogram with exchange fused", lambda: pc.histogram256_u8(u)),
    ("K1 2^25 alone", lambda: ops.reduce_sum_i32(x)),
    ("compaction 2^25 alone", lambda: ops.compact_gt0_i32(x, out, cnt)),
    ("histogram 2^29 alone", lambda: ops.histogram256_u8(u)),
]
# variants interleaved round-robin so clock / thermal drift hits all alike
res = {name: [] for name, _ in rows}
for name, fn in rows:
    timed(fn, iters=10, rounds=1)  # warm
for _ in range(15):
    for name, fn in rows:
        res[name].append(timed(fn, iters=50, rounds=1))
for name, _ in rows:
    v = sorted(res[name])
    print(f"| {name} | {statistics.median(v):.1f} | {v[len(v) // 4]:.1f}-{v[3 * len(v) // 4]:.1f} |",
          flush=True)
assert not pc.failed()
torch.cuda.synchronize()
boxes[0].close()
kboxes[0].close()
