"""Run the acceptance fuzz kernels one by one, printing progress (find hangs)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2112_10034_b200 as wf
from paper_2112_10034_b200.dsl import hybrid_transform, parse_module
cases = json.loads(Path("tests/golden/acceptance_fuzz.json").read_text())["cases"]
start = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = wf.LaunchConfig(grid_size=1, block_size=8, warp_size=4)
gin0 = (np.arange(8) * 5 - 9).astype(np.int32)
t0 = time.time(); bad = []
for seed, src, wg, wo in cases[start:]:
    print("seed", seed, round(time.time() - t0, 1), flush=True)
    k = parse_module(src).kernel()
    mem = wf.DeviceMemory()
    a = mem.alloc(32); mem.write(a, gin0, "i32")
    b = mem.alloc(32); mem.write(b, np.zeros(8, dtype=np.int32), "i32")
    wf.launch(hybrid_transform(k, cfg), cfg, mem, [a, b, 2])
    if mem.host_view(a, "i32").tolist() != wg or mem.host_view(b, "i32").tolist() != wo:
        bad.append(seed)
print("done", round(time.time() - t0, 1), "bad", bad)
