"""K5 per launch, back to back (20 launches between two events), plain vs
WF_FLAG_INPUT_STABLE, rounds interleaved (A B A B ...) so clock / power drift
hits both alike, with the SM clock and throttle reasons sampled meanwhile;
per-GPU shard sizes of the 2^32 job under 1/2/4/8-GPU strong scaling.
usage: python tools/k5_pdl_probe.py [gen]"""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2112_10034_b200 import ops, p2p  # noqa: E402

gen = sys.argv[1] if len(sys.argv) > 1 else "u8_uniform"
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
boxes = p2p.Mailboxes.local(1, dev, cap=256)
pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)


def one(fn, it=20):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / it


for lg in (29, 30, 31, 32):
    u = ops.fill_synthetic(gen, 1 << lg, seed=0)
    torch.cuda.synchronize()
    variants = {"plain": lambda: ops.histogram256_u8(u),
                "pdl": lambda: ops.histogram256_u8(u, input_stable=True),
                "plain_mg": lambda: pc.histogram256_u8(u),
                "pdl_mg": lambda: pc.histogram256_u8(u, input_stable=True)}
    for fn in variants.values():
        one(fn, 3)
    times = {k: [] for k in variants}
    with ClockSampler(0) as clk:
        for _ in range(5):
            for k, fn in variants.items():
                times[k].append(one(fn))
    res = {"gen": gen, "log2n": lg}
    res.update({k + "_us": round(statistics.median(v), 2) for k, v in times.items()})
    res["clocks"] = clk.summary()
    print(json.dumps(res), flush=True)
    del u
torch.cuda.synchronize()
boxes[0].close()
