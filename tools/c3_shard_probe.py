"""Sharded C3 per-rank step at shard sizes (world 1 protocol, peer mailbox of
one rank): pass 1 (K1 + carry exchange, fused) then the scan with the device
carry.  Reports the step, its two passes alone, and a plain copy of the shard.
usage: WF_LIB=... python tools/c3_shard_probe.py [log2n ...]"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, distributed as wd, ops, p2p  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
boxes = p2p.Mailboxes.local(1, dev, cap=256)
pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)


def t(fn, it=30, r=7):
    torch.cuda.synchronize()
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


P1_BLOCK = int(__import__("os").environ.get("WF_P1_BLOCK", "256"))


def step(x, y, flag=False):
    c = pc.reduce_exscan_i32(x, block=P1_BLOCK, input_stable=flag)[:1]
    return ops.scan_inclusive_i32(x, y, carry=c, input_stable=flag)


for lg in [int(v) for v in sys.argv[1:]] or [25, 26, 27]:
    x = ops.fill_synthetic("i32_full", 1 << lg)
    y = torch.empty_like(x)
    res = {"lib": Path(str(_lib.lib_path())).stem, "log2n": lg,
           "step_us": t(lambda: step(x, y)),
           "step_pdl_us": t(lambda: step(x, y, True)),
           "compact_us": t(lambda: pc.compact_gt0_i32(x, y)),
           "compact_pdl_us": t(lambda: pc.compact_gt0_i32(x, y, input_stable=True)),
           "pass1_block": P1_BLOCK,
           "pass1_us": t(lambda: pc.reduce_exscan_i32(x, block=P1_BLOCK)),
           "scan_us": t(lambda: ops.scan_inclusive_i32(x, y)),
           "copy_us": t(lambda: y.copy_(x))}
    want = torch.cumsum(x.to(torch.int64), 0).to(torch.int32)
    res["ok"] = bool(torch.equal(step(x, y), want))
    print(json.dumps(res), flush=True)
    del x, y
boxes[0].close()
