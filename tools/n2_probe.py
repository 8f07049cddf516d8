"""Two ranks on ONE GPU (gloo, torchrun --nproc-per-node 2): time each fused
peer-memory call of the sharded C3/C4/C5 paths and report the timeout flag.
Diagnoses the same-GPU multi-process bench path (contexts time-slice)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2112_10034_b200 import distributed as wd, ops, p2p  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", 0)
n = int(os.environ.get("N_PROBE", str(1 << 27)))
pc, why = p2p.try_peer_collectives(dev)
print(f"rank {rank}: peer {why}", flush=True)
lo, hi = wd.shard_range(n, rank, world)
x = ops.fill_synthetic("i32_full", hi - lo, seed=0, base=lo, device=dev)
y, out = torch.empty_like(x), torch.empty_like(x)
u = ops.fill_synthetic("u8_uniform", hi - lo, seed=0, base=lo, device=dev)
for name, fn in (("scan", lambda: wd.scan_inclusive_i32(x, y, peer=pc)),
                 ("compact", lambda: wd.compact_gt0_i32(x, out, peer=pc)),
                 ("hist", lambda: wd.histogram256_u8(u, peer=pc))):
    for i in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        print(f"rank {rank}: {name} call {i}: {(time.perf_counter() - t) * 1e3:.1f} ms, "
              f"epoch {pc.epoch}, failed {pc.failed()}", flush=True)
# back to back, as bench.py's time_launches issues them (no host sync between)
for name, fn in (("scan", lambda: wd.scan_inclusive_i32(x, y, peer=pc)),
                 ("compact", lambda: wd.compact_gt0_i32(x, out, peer=pc)),
                 ("hist", lambda: wd.histogram256_u8(u, peer=pc))):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(8):
        fn()
    torch.cuda.synchronize()
    print(f"rank {rank}: {name} x8 back to back: {(time.perf_counter() - t) * 1e3:.1f} ms, "
          f"epoch {pc.epoch}, failed {pc.failed()}", flush=True)
dist.destroy_process_group()
