"""Stress the TMEM-parked scan / compaction: many back-to-back launches at
random sizes on one workspace, interleaved with other work on the stream,
each result checked (scan: last element == wrapping sum; compaction: count ==
(x > 0).sum()).  Usage: python tools/stress_tmem.py [iterations]"""
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

torch.cuda.set_device(0)
iters = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 200
rng = random.Random(5)
big = ops.fill_synthetic("i32_full", 1 << 28, seed=3)
out = torch.empty_like(big)
# optional competing work on a second stream (other kernels occupying SMs
# while the persistent TMEM grid launches: not every CTA is resident at once)
other = torch.cuda.Stream() if "--concurrent" in sys.argv else None
f = ops.fill_synthetic("f32_unit", 1 << 28, seed=4) if other else None
t0 = time.time()
for it in range(iters):
    n = rng.choice([1, 7, 8192, 8193, 1 << 20, (1 << 22) + 5, rng.randrange(1, 1 << 28), 1 << 28])
    x = big[:n]
    if other is not None:
        with torch.cuda.stream(other):
            for _ in range(3):
                ops.reduce_sum_f32(f)
    if it % 2 == 0:
        y = ops.scan_inclusive_i32(x, out[:n])
        want = int(ops.reduce_sum_i32(x).item()) & 0xFFFFFFFF
        got = int(y[-1].item()) & 0xFFFFFFFF
        assert got == want, (it, n, got, want)
    else:
        _, cnt = ops.compact_gt0_i32(x, out[:n])
        assert int(cnt.item()) == int((x > 0).sum().item()), (it, n)
    if it % 10 == 0:
        torch.cuda.synchronize()
print(f"stress ok: {iters} launches in {time.time() - t0:.1f} s")
