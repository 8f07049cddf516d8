"""Three K4 launches at the 8-GPU shard size (2^25, 50 %) for an ncu source-level capture."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2112_10034_b200 import ops
torch.cuda.set_device(0)
n = 1 << 25
out = torch.empty(n, dtype=torch.int32, device="cuda")
cnt = torch.empty(1, dtype=torch.int64, device="cuda")
x = ops.fill_synthetic("i32_select", n, seed=0, param=500)
for _ in range(3):
    ops.compact_gt0_i32(x, out, cnt)
torch.cuda.synchronize()
print(int(cnt.item()))
