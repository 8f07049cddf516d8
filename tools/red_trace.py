"""Where does K2's fixed per-launch cost go at shard sizes?  Per-block
globaltimer stamps (variant build -DWF_RED_TRACE=1): block start, block sum
formed (streaming done), the last block's fold done.  Prints, per launch of a
back-to-back sequence, the spread of block starts, the percentiles of the
streaming ends and the fold, relative to the earliest block start, beside the
CUDA-event time of the same launches.
usage: WF_LIB=build/variants/lib_redtrace.so python tools/red_trace.py [log2n] [block]"""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import _lib, ops  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
block = int(sys.argv[2]) if len(sys.argv) > 2 else 512
torch.cuda.set_device(0)
lib = _lib.load()
setter = lib.wf_debug_set_trace_red
setter.argtypes = [ctypes.c_void_p]
x = ops.fill_synthetic("f32_unit", 1 << lg, seed=1)
out = torch.empty(1, dtype=torch.float32, device="cuda")
NL = 6
REC = 4 * 16384 + 8
big = torch.zeros(NL * REC, dtype=torch.int64, device="cuda")
bufs = [big[k * REC:(k + 1) * REC] for k in range(NL)]
for _ in range(5):
    ops.reduce_sum_f32(x, out, block=block)
torch.cuda.synchronize()
ev = [torch.cuda.Event(True) for _ in range(NL + 1)]
# back-to-back: launch k stamps record k (the kernel's own launch counter)
assert setter(big.data_ptr()) == 0
ev[0].record()
for k in range(NL):
    ops.reduce_sum_f32(x, out, block=block)
    ev[k + 1].record()
torch.cuda.synchronize()
assert setter(None) == 0
prev_end = None
for k in range(NL):
    b = bufs[k].cpu()
    nz = int((b[:4 * 16384].view(-1, 4)[:, 1] != 0).sum())
    g = nz
    t = b[: 4 * g].view(g, 4)
    t0 = int(t[:, 0].min())
    st = (t[:, 0] - t0).double() / 1e3
    en = (t[:, 1] - t0).double() / 1e3
    fold = (int(b[4 * g]) - t0) / 1e3
    q = torch.tensor([0.0, 0.5, 0.9, 0.99, 1.0], dtype=torch.double)
    row = {"launch": k, "grid": g, "event_us": round(ev[k].elapsed_time(ev[k + 1]) * 1e3, 1),
           "start_spread_us": round(float(st.max()), 2),
           "stream_end_pcts_us": [round(float(v), 2) for v in torch.quantile(en, q)],
           "fold_done_us": round(fold, 2),
           "gap_from_prev_fold_us": None if prev_end is None else round((t0 - prev_end) / 1e3, 2)}
    prev_end = int(b[4 * g])
    print(json.dumps(row), flush=True)
