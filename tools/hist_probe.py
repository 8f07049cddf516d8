import sys, statistics, json
sys.path.insert(0, '.')
import torch
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)
n = 1 << 32
for gen in ("u8_uniform", "u8_const", "u8_geom"):
    x = ops.fill_synthetic(gen, n, seed=4)
    ops.histogram256_u8(x); torch.cuda.synchronize()
    v = []
    for _ in range(5):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(10): ops.histogram256_u8(x)
        b.record(); b.synchronize(); v.append(a.elapsed_time(b) * 100)
    bins = ops.histogram256_u8(x).cpu()
    print(json.dumps({"gen": gen, "us": round(statistics.median(v), 1), "all": [round(t,1) for t in v], "maxbin_frac": float(bins.max()) / n}))
    del x
