"""Run the acceptance fuzz kernels; print every failing seed with its source
and generated CUDA (debugging aid)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2112_10034_b200 as wf
from paper_2112_10034_b200.dsl import hybrid_transform, parse_module
cases = json.loads(Path("tests/golden/acceptance_fuzz.json").read_text())["cases"]
cfg = wf.LaunchConfig(grid_size=1, block_size=8, warp_size=4)
gin0 = (np.arange(8) * 5 - 9).astype(np.int32)
shown = 0
for seed, src, wg, wo in cases:
    k = parse_module(src).kernel()
    mem = wf.DeviceMemory()
    a = mem.alloc(32); mem.write(a, gin0, "i32")
    b = mem.alloc(32); mem.write(b, np.zeros(8, dtype=np.int32), "i32")
    prog = hybrid_transform(k, cfg)
    try:
        wf.launch(prog, cfg, mem, [a, b, 2])
        ok = mem.host_view(a, "i32").tolist() == wg and mem.host_view(b, "i32").tolist() == wo
        err = ""
    except Exception as e:
        ok, err = False, repr(e)
    if not ok:
        print("=== seed", seed, err, "\nwant", wg, wo, "\ngot", mem.host_view(a, "i32").tolist(),
              mem.host_view(b, "i32").tolist())
        if shown < 3:
            print(src); print(prog.source)
        shown += 1
print("done")
