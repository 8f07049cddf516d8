import sys, torch, statistics
sys.path.insert(0, ".")
from paper_2112_10034_b200 import ops
def t(fn, it=50, r=9):
    fn(); torch.cuda.synchronize(); v=[]
    for _ in range(r):
        a,b=torch.cuda.Event(True),torch.cuda.Event(True); a.record()
        for _ in range(it): fn()
        b.record(); b.synchronize(); v.append(a.elapsed_time(b)*1e3/it)
    return statistics.median(v)
for lg in (24, 25, 26, 28):
    x = ops.fill_synthetic("i32_full", 1 << lg); y = torch.empty_like(x)
    print(lg, "scan", round(t(lambda: ops.scan_inclusive_i32(x, y)), 1), "copy", round(t(lambda: y.copy_(x)), 1), "K1", round(t(lambda: ops.reduce_sum_i32(x)), 1))
