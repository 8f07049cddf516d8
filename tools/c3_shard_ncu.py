"""One launch each at the 8-GPU shard (2^25 int32, world-1 mailbox) of: the
block-cyclic single-pass scan, and reduce-then-scan (pass 1 + scan with
carry), for an ncu capture of their DRAM bytes (8 vs 12 B/elem)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops, p2p  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
boxes = p2p.Mailboxes.local(1, dev, cap=256)
pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)
n = 1 << 25
x = ops.fill_synthetic("i32_full", n, seed=0)
y = torch.empty_like(x)
torch.cuda.synchronize()
pc.scan_inclusive_i32_cyclic(x, y, 1 << 22, n >> 22)          # block-cyclic, single pass
torch.cuda.synchronize()
c = pc.reduce_exscan_i32(x)[:1]                                # reduce-then-scan: pass 1
ops.scan_inclusive_i32(x, y, carry=c)                          # ... and the scan
torch.cuda.synchronize()
assert not pc.failed()
boxes[0].close()
print("ok")
