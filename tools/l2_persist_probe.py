"""Sharded C3 per-rank step (world-1 protocol, as tools/c3_shard_probe.py)
under the L2 persisting set-aside: does pass 1's tail of reads (the shard's
head, read last because pass 1 streams backwards) survive in L2 until the
scan reads it first, when L2 lines can be PERSISTING instead of merely
evict_last-hinted?

Modes per shard size:
  base      current library, persisting limit 0 (the shipped behaviour)
  limit     cudaLimitPersistingL2CacheSize = max (evict_last lines may
            count as persisting)
  window W  limit = max and an accessPolicyWindow over the shard's first W
            bytes on the stream during pass 1 (hitProp persisting), and over
            the same bytes with hitProp normal during the scan (demotes the
            lines as they are consumed, so nothing persists into the next
            step)
Each mode is timed back to back (30 steps) and with a 256 MiB L2 flush
between steps (events around each step only).
usage: WF_LIB=... python tools/l2_persist_probe.py [log2n ...]"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

from paper_2112_10034_b200 import _lib, ops, p2p  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
boxes = p2p.Mailboxes.local(1, dev, cap=256)
pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)
stream = torch.cuda.current_stream()
h = stream.cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

err, maxp = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
err, maxw = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0)
err, l2 = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0)
print(json.dumps({"lib": Path(str(_lib.lib_path())).stem, "l2_bytes": l2,
                  "max_persisting_bytes": maxp, "max_window_bytes": maxw}), flush=True)


def set_limit(b):
    (e,) = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, b)
    assert e == rt.cudaError_t.cudaSuccess, e


def window(base, nbytes, prop):
    v = rt.cudaStreamAttrValue()
    w = v.accessPolicyWindow
    w.base_ptr = base
    w.num_bytes = nbytes
    w.hitRatio = 1.0
    w.hitProp = prop
    w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    v.accessPolicyWindow = w
    (e,) = rt.cudaStreamSetAttribute(h, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, v)
    assert e == rt.cudaError_t.cudaSuccess, e


def no_window():
    window(0, 0, rt.cudaAccessProperty.cudaAccessPropertyNormal)


def timed(fn, it=30, r=5):
    fn()
    torch.cuda.synchronize()
    v = []
    for _ in range(r):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(it):
            fn()
        b.record()
        b.synchronize()
        v.append(a.elapsed_time(b) * 1e3 / it)
    return round(statistics.median(v), 1)


def timed_flushed(fn, it=20):
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(it)]
    for a, b in ev:
        flush.fill_(1)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return round(statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev), 1)


for lg in [int(v) for v in sys.argv[1:]] or [25, 26]:
    x = ops.fill_synthetic("i32_full", 1 << lg)
    y = torch.empty_like(x)
    want = torch.cumsum(x.to(torch.int64), 0).to(torch.int32)

    def step_plain():
        c = pc.reduce_exscan_i32(x)[:1]
        ops.scan_inclusive_i32(x, y, carry=c)

    modes = [("base", 0, None), ("limit", maxp, None)]
    for mb in (32, 48, 64, 80, 96, 112):
        if (mb << 20) <= min(maxp, maxw, x.numel() * 4):
            modes.append((f"window{mb}", maxp, mb << 20))
    for name, lim, wb in modes:
        set_limit(lim)
        if wb is None:
            fn = step_plain
        else:
            def fn(wb=wb):
                window(x.data_ptr(), wb, rt.cudaAccessProperty.cudaAccessPropertyPersisting)
                c = pc.reduce_exscan_i32(x)[:1]
                window(x.data_ptr(), wb, rt.cudaAccessProperty.cudaAccessPropertyNormal)
                ops.scan_inclusive_i32(x, y, carry=c)
                no_window()
        res = {"log2n": lg, "mode": name, "limit": lim,
               "step_us": timed(fn), "step_flushed_us": timed_flushed(fn)}
        fn()
        torch.cuda.synchronize()
        res["ok"] = bool(torch.equal(y, want))
        print(json.dumps(res), flush=True)
        no_window()
        set_limit(0)
        rt.cudaCtxResetPersistingL2Cache()
    res = {"log2n": lg, "scan_only_flushed_us": timed_flushed(lambda: ops.scan_inclusive_i32(x, y)),
           "pass1_only_flushed_us": timed_flushed(lambda: pc.reduce_exscan_i32(x)),
           "copy_flushed_us": timed_flushed(lambda: y.copy_(x))}
    print(json.dumps(res), flush=True)
    del x, y, want
boxes[0].close()
