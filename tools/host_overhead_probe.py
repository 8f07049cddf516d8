"""Per-call host cost of the tensor-level ops wrappers (GPU box)."""
import time

import torch

from paper_2112_10034_b200 import _lib, ops


def per_call(fn, iters=20000):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / iters * 1e6


x = torch.ones(1 << 20, dtype=torch.int32, device="cuda")
out = torch.empty(1, dtype=torch.int32, device="cuda")
lib = _lib.load()
ws = ops.workspace(_lib.OP_REDUCE_SUM_I32, x.numel(), x.device)
s = torch.cuda.current_stream().cuda_stream
xp, op, wp, wn, n = x.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), x.numel()
rows = {
    "ops.reduce_sum_i32": lambda: ops.reduce_sum_i32(x, out),
    "ctypes direct": lambda: lib.wf_reduce_sum_i32(xp, n, op, 256, 0, wp, wn, s),
    "current_stream().cuda_stream": lambda: torch.cuda.current_stream().cuda_stream,
    "_cuda_getCurrentRawStream": lambda: torch._C._cuda_getCurrentRawStream(0),
    "workspace()": lambda: ops.workspace(_lib.OP_REDUCE_SUM_I32, n, x.device),
    "wf_workspace_bytes": lambda: lib.wf_workspace_bytes(1, n, 256),
    "_require_cuda": lambda: ops._require_cuda(x, torch.int32, "x"),
    "x.device": lambda: x.device,
    "x.data_ptr()": lambda: x.data_ptr(),
    "torch x.add_(0)": lambda: x.add_(0),
    "ops.scan (2^20)": lambda: ops.scan_inclusive_i32(x, torch.empty_like(x)),
    "ops.histogram": lambda: ops.histogram256_u8(x.view(torch.uint8)),
}
for k, f in rows.items():
    print(f"{k:32s} {per_call(f, 5000 if k.startswith('ops.scan') else 20000):7.2f} us")
print(f"{'torch.cuda.current_device()':32s} {per_call(torch.cuda.current_device):7.2f} us")
print(f"{'ops._stream_handle()':32s} {per_call(ops._stream_handle):7.2f} us")
