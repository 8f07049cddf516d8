"""K2 per launch, back to back (20 launches between two events, median of 5
rounds), plain vs WF_FLAG_INPUT_STABLE (programmatic dependent launch), at
the per-GPU shard sizes of the 2^30 job under 1/2/4/8-GPU strong scaling.
usage: python tools/k2_pdl_probe.py"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops, p2p  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
boxes = p2p.Mailboxes.local(1, dev)
pr = p2p.PeerReducer(boxes[0], 0, 1)


def t(fn, it=20, r=5):
    for _ in range(3):
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
    return round(statistics.median(v), 2)


for lg in [int(v) for v in sys.argv[1:]] or (27, 28, 29, 30):
    x = ops.fill_synthetic("f32_unit", 1 << lg, seed=1)
    torch.cuda.synchronize()
    for block in (256, 512, 1024):
        res = {"log2n": lg, "block": block}
        for name, st in (("plain", False), ("pdl", True)):
            res[name + "_us"] = t(lambda: ops.reduce_sum_f32(x, block=block, input_stable=st))
            res[name + "_mg_us"] = t(lambda: pr.reduce_sum_f32(x, block=block, input_stable=st))
        res["pdl_gbs"] = round(4 * x.numel() / res["pdl_us"] / 1e3, 1)
        print(json.dumps(res), flush=True)
    del x
torch.cuda.synchronize()
boxes[0].close()
