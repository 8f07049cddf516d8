import sys, torch
sys.path.insert(0, ".")
from paper_2112_10034_b200 import ops, p2p, distributed as wd
dev = torch.device("cuda", 0)
world = 2
for which in ("k1", "hist", "exscan"):
    boxes = p2p.Mailboxes.local(world, dev, cap=256)
    pcs = [p2p.PeerCollectives(boxes[r], r, world, 256, dev) for r in range(world)]
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    xs = [ops.fill_synthetic("i32_full", 1 << 22, seed=5, base=r << 22) for r in range(world)]
    us = [ops.fill_synthetic("u8_uniform", 1 << 24, seed=6, base=r << 24) for r in range(world)]
    torch.cuda.synchronize()
    outs = []
    for r in range(world):
        with torch.cuda.stream(streams[r]):
            if which == "k1":
                outs.append(pcs[r].reduce_exscan_i32(xs[r], stream=streams[r]))
            elif which == "hist":
                outs.append(pcs[r].histogram256_u8(us[r], stream=streams[r]))
            else:
                outs.append(pcs[r].exscan_u64(torch.tensor([r + 1], device=dev), stream=streams[r]))
    torch.cuda.synchronize()
    print(which, [pc.failed() for pc in pcs], [o[:4].tolist() for o in outs], flush=True)
    boxes[0].close()
