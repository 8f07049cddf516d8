"""C1 (2^20 int32 reduction) latency vs block/grid: flushed-L2 CUDA-event time
per launch, plus the steady-state time per launch inside a CUDA graph of 50
back-to-back launches (no host overhead, L2 warm)."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

torch.cuda.set_device(0)
x = ops.fill_synthetic("i32_full", 1 << 20)
out = torch.empty(1, dtype=torch.int32, device="cuda")
fb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
want = int(x.to(torch.int64).sum().item()) & 0xFFFFFFFF
for block in (256, 512, 1024):
    for grid in (0, 32, 64, 128, 148, 256, 296):
        if grid and grid * block * 16 > (1 << 20) * 4:
            continue
        f = lambda: ops.reduce_sum_i32(x, out, block=block, grid=grid)
        for _ in range(3):
            f()
        ok = (int(out.item()) & 0xFFFFFFFF) == want
        ts = []
        for _ in range(30):
            fb.fill_(1)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); f(); e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            f()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=st):
                for _ in range(50):
                    f()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.replay(); e.record(); torch.cuda.synchronize()
        print(json.dumps({"block": block, "grid": grid, "ok": ok,
                          "flushed_us": round(statistics.median(ts), 2),
                          "graph_us_per_launch": round(s.elapsed_time(e) * 1e3 / 50, 2)}))
