"""K2 time vs shard size (the per-GPU work at 1/2/4/8 GPUs under strong
scaling of the 2^30 job), plain and with the fused exchange (world 1)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops, p2p  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
boxes = p2p.Mailboxes.local(1, dev)
pr = p2p.PeerReducer(boxes[0], 0, 1)
for lg in (27, 30):
    x = ops.fill_synthetic("f32_unit", 1 << lg, seed=1)
    res = {"n": f"2^{lg}"}
    for name, fn in (("k2", lambda: ops.reduce_sum_f32(x)), ("k2_fused_w1", lambda: pr.reduce_sum_f32(x))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            fn()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3 / 20
        res[name + "_us"] = round(us, 2)
        res[name + "_gbs"] = round(4 * (1 << lg) / us / 1e3, 1)
    print(json.dumps(res), flush=True)
    del x
torch.cuda.synchronize()
boxes[0].close()
