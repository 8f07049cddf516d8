"""Block-cyclic scan with `world` ranks as concurrent kernels on ONE GPU
(grids of 148/world CTAs, every rank on its own stream), total 2^28: if the
rounds' cross-rank waits serialised the ranks, the whole call would take a
multiple of the one-rank time; sharing one GPU's bandwidth, it should take
about the same as one rank scanning everything.  usage: python
tools/cyclic_inprocess_probe.py"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import distributed as wd, ops, p2p  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
n = 1 << 28
full = ops.fill_synthetic("i32_full", n, seed=5)
want = torch.cumsum(full.to(torch.int64), 0).to(torch.int32)
for world in (1, 2, 4, 8):
    # a round must fit a rank's pipeline (12 tiles per CTA): with 148 / world
    # CTAs per rank here, rounds shrink with the world (a whole GPU per rank
    # holds 1776 tiles: 2^22-element rounds, 512 tiles, fit 3x over)
    round_elems = (1 << 22) // world
    boxes = p2p.Mailboxes.local(world, dev, cap=256)
    pcs = [p2p.PeerCollectives(boxes[r], r, world, 256, dev) for r in range(world)]
    lay = [wd.cyclic_rounds(n, r, world, round_elems) for r in range(world)]
    rounds = lay[0][0]
    xs = [torch.cat([full[s:s + m] for s, m in lay[r][1]]) for r in range(world)]
    ys = [torch.empty_like(x) for x in xs]
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    cap = 148 // world

    def call():
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                pcs[r].scan_inclusive_i32_cyclic(xs[r], ys[r], round_elems, rounds,
                                                 max_grid=cap, stream=streams[r])
        torch.cuda.synchronize()

    call()
    ts = []
    for _ in range(7):
        a = torch.cuda.Event(True)
        b = torch.cuda.Event(True)
        a.record()
        call()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ok = all(torch.equal(ys[r], torch.cat([want[s:s + m] for s, m in lay[r][1]]))
             for r in range(world))
    print(json.dumps({"world": world, "ctas_per_rank": cap, "round_elems": round_elems, "call_us": round(statistics.median(ts), 1),
                      "ok": ok, "failed": any(pc.failed() for pc in pcs)}), flush=True)
    torch.cuda.synchronize()
    boxes[0].close()
    del xs, ys
