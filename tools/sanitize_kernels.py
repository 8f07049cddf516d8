"""Small invocation of every hot-path kernel for compute-sanitizer
(memcheck / racecheck / synccheck):  compute-sanitizer --tool racecheck
python tools/sanitize_kernels.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

torch.cuda.set_device(0)
n = 8192 * 300 + 123  # > one persistent wave of tiles, ragged tail
x = ops.fill_synthetic("i32_full", n, seed=1)
f = ops.fill_synthetic("f32_unit", n, seed=2)
u = ops.fill_synthetic("u8_uniform", 4 * n + 5, seed=3)
r = [ops.reduce_sum_i32(x), ops.reduce_sum_f32(f), ops.scan_inclusive_i32(x),
     ops.compact_gt0_i32(x)[1], ops.histogram256_u8(u),
     ops.scan_inclusive_i32(x[1:]), ops.compact_gt0_i32(x[3:])[1]]
a = torch.arange(96, dtype=torch.int32, device="cuda")
for kind in ("shfl_down", "shfl_up", "shfl_xor", "shfl_idx", "vote_all", "vote_any", "ballot", "reduce_add"):
    r.append(ops.warp_collective(kind, a, operand=3, block=96))
# the reference's own formulations (dsl/patterns.py native kernels)
from paper_2112_10034_b200.dsl import patterns  # noqa: E402
st = torch.cuda.current_stream().cuda_stream
for name, sym, nn in (("warp_partials_sum_i32", "wf_warp_partials_sum_i32", "n"),
                      ("warp_partials_sum_f32", "wf_warp_partials_sum_f32", "n")):
    pat = patterns.NativePattern(name, sym, "a", "out", nn)
    cfg = type("C", (), {"grid_size": 37, "block_size": 96, "warp_size": 32})()
    o = torch.zeros(37 * 3, dtype=torch.int32, device="cuda")
    pat.run(cfg, {"a": x if "i32" in name else f, "out": o, "n": n}, st)
    r.append(o)
pat = patterns.NativePattern("warp_prefix32_i32", "wf_warp_prefix32_i32", "a", "out")
cfg = type("C", (), {"grid_size": 300, "block_size": 256, "warp_size": 32})()
o = torch.zeros(300 * 256, dtype=torch.int32, device="cuda")
pat.run(cfg, {"a": x, "out": o}, st)
pat.run(cfg, {"a": x[1:], "out": o}, st)
r.append(o)
# the fused multi-GPU forms (world 1: own mailbox; the peer stores and the
# flag/epoch protocol still run)
from paper_2112_10034_b200 import p2p  # noqa: E402
dev = torch.device("cuda", 0)
boxes = p2p.Mailboxes.local(1, dev, cap=256)
pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)
r += [pc.reduce_exscan_i32(x), pc.compact_gt0_i32(x)[1], pc.histogram256_u8(u),
      pc.exscan_u64(torch.ones(1, dtype=torch.int64, device=dev))]
kboxes = p2p.Mailboxes.local(1, dev)
r.append(p2p.PeerReducer(kboxes[0], 0, 1).reduce_sum_f32(f))
# WF_FLAG_INPUT_STABLE chains (programmatic dependent launches: each launch
# starts while its predecessor drains, griddepcontrol.wait before the workspace)
torch.cuda.synchronize()
y = torch.empty_like(x)
for _ in range(3):
    r.append(ops.reduce_sum_f32(f, input_stable=True))
    r.append(ops.histogram256_u8(u, input_stable=True))
    ops.scan_inclusive_i32(x, y, input_stable=True)
    r.append(ops.compact_gt0_i32(x, input_stable=True)[1])
    r.append(pc.reduce_exscan_i32(x, input_stable=True))
    ops.scan_inclusive_i32(x, y, carry=r[-1][:1], input_stable=True)
    r.append(pc.compact_gt0_i32(x, input_stable=True)[1])
    r.append(pc.histogram256_u8(u, input_stable=True))
r.append(y)
# the block-cyclic single-pass scan (world 1: its totaler, sweeper and mailbox
# rounds execute), plain and dependent, rounds of 16 tiles
xc = ops.fill_synthetic("i32_full", 8192 * 16 * 5 + 8192 * 3, seed=9)
yc = torch.empty_like(xc)
for flag in (False, True):
    pc.scan_inclusive_i32_cyclic(xc, yc, 8192 * 16, 6, input_stable=flag)
r.append(yc)
torch.cuda.synchronize()
assert torch.equal(yc, torch.cumsum(xc.to(torch.int64), 0).to(torch.int32))
assert not pc.failed()
boxes[0].close()
kboxes[0].close()
print("ok", [int(t.reshape(-1)[0].item()) if t.dtype != torch.float32 else float(t[0]) for t in r[:5]])
