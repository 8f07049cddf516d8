import sys, json, statistics
sys.path.insert(0, '.')
import torch
from paper_2112_10034_b200 import ops, p2p, distributed as wd
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
boxes = p2p.Mailboxes.local(1, dev, cap=256)
pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)
def one(fn, it=20):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it): fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) * 1e3 / it
for lg in (25, 26, 27, 28):
    x = ops.fill_synthetic("i32_full", 1 << lg, seed=0)
    y = torch.empty_like(x)
    res = {"log2n": lg}
    fns = {}
    for re in (20, 21, 22, 23):
        R = -(-x.numel() // (1 << re))
        fns[f"cyclic_r2^{re}"] = (lambda re=re, R=R: pc.scan_inclusive_i32_cyclic(x, y, 1 << re, R, input_stable=True))
    fns["plain_pdl"] = lambda: ops.scan_inclusive_i32(x, y, input_stable=True)
    def two():
        c = pc.reduce_exscan_i32(x, input_stable=True)[:1]
        ops.scan_inclusive_i32(x, y, carry=c, input_stable=True)
    fns["reduce_then_scan"] = two
    torch.cuda.synchronize()
    for f in fns.values(): f()
    t = {k: [] for k in fns}
    for _ in range(5):
        for k, f in fns.items():
            torch.cuda.synchronize(); t[k].append(one(f))
    res.update({k: round(statistics.median(v), 1) for k, v in t.items()})
    pc.scan_inclusive_i32_cyclic(x, y, 1 << 22, -(-x.numel() // (1 << 22)))
    res["ok"] = bool(torch.equal(y, torch.cumsum(x.to(torch.int64), 0).to(torch.int32)))
    print(json.dumps(res), flush=True)
    del x, y
assert not pc.failed()
boxes[0].close()
