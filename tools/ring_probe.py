"""Host-buffer scan (C3 e2e) vs the PCIe ceiling: where does the ring lose?
Times (host clock, median of 5): one concurrent pinned H2D + D2H of 1 GiB
each; the same bytes as a chunked ring of plain copies (H2D stream, D2H
stream waiting on each chunk's H2D) at several chunk sizes; and
ops.scan_inclusive_i32_host.  usage: python tools/ring_probe.py"""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2112_10034_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
n = 1 << 28
x = ops.fill_synthetic("i32_full", n)
hin = torch.empty(n, dtype=torch.int32, pin_memory=True)
hin.copy_(x)
hout = torch.empty(n, dtype=torch.int32, pin_memory=True)
d = torch.empty_like(x)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def med(fn, r=5):
    fn()
    torch.cuda.synchronize()
    v = []
    for _ in range(r):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        v.append(time.perf_counter() - t)
    return round(statistics.median(v) * 1e3, 3)


def link():
    with torch.cuda.stream(s1):
        d.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(x, non_blocking=True)


def ring(chunk_elems):
    def fn():
        for c in range(0, n, chunk_elems):
            e = torch.cuda.Event()
            with torch.cuda.stream(s1):
                d[c:c + chunk_elems].copy_(hin[c:c + chunk_elems], non_blocking=True)
                e.record(s1)
            s2.wait_event(e)
            with torch.cuda.stream(s2):
                hout[c:c + chunk_elems].copy_(d[c:c + chunk_elems], non_blocking=True)
    return fn


s3 = torch.cuda.Stream()


def ring_kernel(chunk_elems):
    """the same ring with a torch kernel (in-place +0 on the chunk, one HBM
    read + write pass) between each chunk's H2D and its D2H, on a third
    stream: does any kernel in the ring cost the copies time?"""
    def fn():
        for c in range(0, n, chunk_elems):
            e1, e2 = torch.cuda.Event(), torch.cuda.Event()
            with torch.cuda.stream(s1):
                d[c:c + chunk_elems].copy_(hin[c:c + chunk_elems], non_blocking=True)
                e1.record(s1)
            s3.wait_event(e1)
            with torch.cuda.stream(s3):
                d[c:c + chunk_elems].add_(0)
                e2.record(s3)
            s2.wait_event(e2)
            with torch.cuda.stream(s2):
                hout[c:c + chunk_elems].copy_(d[c:c + chunk_elems], non_blocking=True)
    return fn


def h2d_only():
    d.copy_(hin, non_blocking=True)


def d2h_only():
    hout.copy_(x, non_blocking=True)


res = {"link_ms": med(link), "h2d_only_ms": med(h2d_only), "d2h_only_ms": med(d2h_only)}
for mb in (1, 2, 4, 8, 16, 32, 64):
    res[f"ring_{mb}MiB_ms"] = med(ring((mb << 20) // 4))
res["ring_16MiB_torch_kernel_ms"] = med(ring_kernel((16 << 20) // 4))
res["scan_host_ms"] = med(lambda: ops.scan_inclusive_i32_host(hin, hout, device=dev))
res["scan_host_ok"] = bool(torch.equal(hout, ops.scan_inclusive_i32(x).cpu()))
res["frac_of_link"] = round(res["link_ms"] / res["scan_host_ms"], 4)
print(json.dumps(res), flush=True)
