"""One K4 launch at 2^28 for each of 0 %, 1 % and 50 % selectivity (for an
ncu --set full capture of tile_tmem_kernel<1, 0>)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

torch.cuda.set_device(0)
n = 1 << 28
out = torch.empty(n, dtype=torch.int32, device="cuda")
cnt = torch.empty(1, dtype=torch.int64, device="cuda")
for p in (0, 10, 500):
    x = ops.fill_synthetic("i32_select", n, seed=0, param=p)
    ops.compact_gt0_i32(x, out, cnt)
    torch.cuda.synchronize()
    print(p, int(cnt.item()))
