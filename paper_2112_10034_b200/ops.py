"""Tensor-level API of the five warp-primitive kernels (K1–K5) and the warp
collectives (P), each a thin call into the C ABI.

These are the B200 replacements for what the reference computes by running
a DSL kernel through ``launch(hybrid_transform(...))`` (runtime/launch.py:90,
passes/pipeline.py:103) on CPU workers.  Inputs/outputs are CUDA tensors
(PyTorch is only the allocator and stream provider); work is enqueued on the
current torch stream and is asynchronous — call ``torch.cuda.synchronize()``
or use :func:`paper_2112_10034_b200.launch` for the reference's join
semantics.
"""

from __future__ import annotations

import contextlib
import threading

import torch

from . import _lib
from ._lib import check
from .errors import ConfigError, LaunchError

REDUCE_BLOCKS = (128, 256, 512, 1024)

_ws_lock = threading.Lock()
_ws_cache: dict = {}


# The raw handle of the current stream without building a torch.cuda.Stream
# object: 0.1 us instead of 3.3 us per call on the B200 box
# (tools/host_overhead_probe.py), a third of a small op's host cost.
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_handle(stream=None) -> int:
    if stream is not None:
        return int(stream.cuda_stream)
    if _raw_stream is not None:
        return int(_raw_stream(torch.cuda.current_device()))
    return int(torch.cuda.current_stream().cuda_stream)


def _on(device) -> contextlib.AbstractContextManager:
    """Make ``device`` current for one launch: the C ABI launches on the
    current device and stream, so a tensor on another GPU must switch first
    (a no-op context when it is already current)."""
    idx = device.index if isinstance(device, torch.device) else int(device)
    if idx is None or idx == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(idx)


def workspace(op: int, n: int, device: torch.device, stream=None) -> torch.Tensor:
    """Zero-initialised scratch for ``op`` (cached per device/op/stream; the
    kernels leave it reusable, so it is zeroed only when (re)allocated)."""
    lib = _lib.load()
    need = int(lib.wf_workspace_bytes(op, n, 256))
    if need == 0:
        return None
    key = (device.index, op, _stream_handle(stream))
    with _ws_lock:
        ws = _ws_cache.get(key)
        if ws is None or ws.numel() < need:
            size = max(need, 2 * ws.numel() if ws is not None else 0)
            ws = torch.zeros(size + 256, dtype=torch.uint8, device=device)
            off = (-ws.data_ptr()) % 256
            ws = ws[off:off + size]  # zero fill is ordered before use on this stream
            _ws_cache[key] = ws
    return ws


def release_workspaces() -> None:
    with _ws_lock:
        _ws_cache.clear()


def _require_cuda(t: torch.Tensor, dtype, name: str) -> None:
    if not isinstance(t, torch.Tensor):
        raise LaunchError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise LaunchError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise LaunchError(f"{name} must have dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise LaunchError(f"{name} must be contiguous")


def _check_block(block: int) -> None:
    if block not in REDUCE_BLOCKS:
        raise ConfigError(f"block size must be one of {REDUCE_BLOCKS}, got {block}")


# ---- K1 / K2 -------------------------------------------------------------

def reduce_sum_i32(x: torch.Tensor, out: torch.Tensor | None = None, block: int = 256,
                   grid: int = 0) -> torch.Tensor:
    """Wrapping int32 sum of ``x`` into ``out[0]`` (K1)."""
    _require_cuda(x, torch.int32, "x")
    _check_block(block)
    if out is None:
        out = torch.empty(1, dtype=torch.int32, device=x.device)
    _require_cuda(out, torch.int32, "out")
    with _on(x.device):
        ws = workspace(_lib.OP_REDUCE_SUM_I32, x.numel(), x.device)
        check(_lib.load().wf_reduce_sum_i32(x.data_ptr(), x.numel(), out.data_ptr(), block, grid,
                                            ws.data_ptr(), ws.numel(), _stream_handle()),
              "reduce_sum_i32")
    return out


def reduce_sum_f32(x: torch.Tensor, out: torch.Tensor | None = None, block: int = 256,
                   grid: int = 0, input_stable: bool = False) -> torch.Tensor:
    """fp32 sum of ``x`` into ``out[0]`` with a fixed association order (K2).

    ``input_stable=True`` is the caller's promise that the kernel issued just
    before on the current stream does not write ``x`` (e.g. the previous call
    of a loop over the same input): the launch then overlaps that kernel's
    tail (``WF_FLAG_INPUT_STABLE``, programmatic dependent launch).  Same
    result bits either way."""
    _require_cuda(x, torch.float32, "x")
    _check_block(block)
    if out is None:
        out = torch.empty(1, dtype=torch.float32, device=x.device)
    _require_cuda(out, torch.float32, "out")
    with _on(x.device):
        ws = workspace(_lib.OP_REDUCE_SUM_F32, x.numel(), x.device)
        check(_lib.load().wf_reduce_sum_f32_ex(x.data_ptr(), x.numel(), out.data_ptr(), block,
                                               grid, ws.data_ptr(), ws.numel(),
                                               _lib.FLAG_INPUT_STABLE if input_stable else 0,
                                               _stream_handle()),
              "reduce_sum_f32")
    return out


def fold(vals: torch.Tensor, count: int | None = None,
         out: torch.Tensor | None = None) -> torch.Tensor:
    """Fixed-order device fold of ``vals[:count]`` (cross-GPU partial combine)."""
    count = vals.numel() if count is None else int(count)
    lib = _lib.load()
    fns = {torch.float32: lib.wf_fold_f32, torch.int32: lib.wf_fold_i32,
           torch.int64: lib.wf_fold_u64}
    if vals.dtype not in fns:
        raise LaunchError(f"fold supports float32/int32/int64, got {vals.dtype}")
    _require_cuda(vals, vals.dtype, "vals")
    if out is None:
        out = torch.empty(1, dtype=vals.dtype, device=vals.device)
    with _on(vals.device):
        check(fns[vals.dtype](vals.data_ptr(), count, out.data_ptr(), _stream_handle()), "fold")
    return out


# ---- K3 / K4 / K5 --------------------------------------------------------

def scan_inclusive_i32(x: torch.Tensor, out: torch.Tensor | None = None,
                       carry: torch.Tensor | None = None,
                       input_stable: bool = False) -> torch.Tensor:
    """Inclusive wrapping prefix sum (K3); ``carry`` (device int32[1]) is added
    to every output (cross-GPU carry-in).  ``out`` may be ``x`` (in place).
    ``input_stable``: WF_FLAG_INPUT_STABLE (the kernel issued just before on
    the stream does not write ``x``; ``carry`` may be its output)."""
    _require_cuda(x, torch.int32, "x")
    if out is None:
        out = torch.empty_like(x)
    _require_cuda(out, torch.int32, "out")
    if out.numel() < x.numel():
        raise LaunchError(f"out holds {out.numel()} elements, need {x.numel()}")
    cptr = None
    if carry is not None:
        _require_cuda(carry, torch.int32, "carry")
        cptr = carry.data_ptr()
    with _on(x.device):
        ws = workspace(_lib.OP_SCAN_INCLUSIVE_I32, x.numel(), x.device)
        check(_lib.load().wf_scan_inclusive_i32_ex(x.data_ptr(), out.data_ptr(), x.numel(), cptr,
                                                   ws.data_ptr(), ws.numel(),
                                                   _lib.FLAG_INPUT_STABLE if input_stable else 0,
                                                   _stream_handle()),
              "scan_inclusive_i32")
    return out


def compact_gt0_i32(x: torch.Tensor, out: torch.Tensor | None = None,
                    count: torch.Tensor | None = None, input_stable: bool = False):
    """Order-preserving ``x[x > 0]`` (K4).  Returns ``(out, count)`` where
    ``out`` has capacity ``x.numel()`` and ``count`` is a device int64[1]
    (bit-identical to the C ABI's uint64).  ``input_stable``:
    WF_FLAG_INPUT_STABLE."""
    _require_cuda(x, torch.int32, "x")
    if out is None:
        out = torch.empty_like(x)
    _require_cuda(out, torch.int32, "out")
    if out.numel() < x.numel():
        raise LaunchError(f"out holds {out.numel()} elements, need {x.numel()}")
    if count is None:
        count = torch.empty(1, dtype=torch.int64, device=x.device)
    _require_cuda(count, torch.int64, "count")
    with _on(x.device):
        ws = workspace(_lib.OP_COMPACT_GT0_I32, x.numel(), x.device)
        check(_lib.load().wf_compact_gt0_i32_ex(x.data_ptr(), x.numel(), out.data_ptr(),
                                                count.data_ptr(), ws.data_ptr(), ws.numel(),
                                                _lib.FLAG_INPUT_STABLE if input_stable else 0,
                                                _stream_handle()),
              "compact_gt0_i32")
    return out, count


def histogram256_u8(x: torch.Tensor, bins: torch.Tensor | None = None,
                    grid: int = 0, input_stable: bool = False) -> torch.Tensor:
    """256-bin byte histogram (K5) as a device int64[256] (== uint64 bits).
    ``input_stable``: as ``reduce_sum_f32`` (WF_FLAG_INPUT_STABLE)."""
    _require_cuda(x, torch.uint8, "x")
    if bins is None:
        bins = torch.empty(256, dtype=torch.int64, device=x.device)
    _require_cuda(bins, torch.int64, "bins")
    if bins.numel() < 256:
        raise LaunchError("bins must hold 256 counters")
    with _on(x.device):
        ws = workspace(_lib.OP_HISTOGRAM256_U8, x.numel(), x.device)
        check(_lib.load().wf_histogram256_u8_ex(x.data_ptr(), x.numel(), bins.data_ptr(), grid,
                                                ws.data_ptr(), ws.numel(),
                                                _lib.FLAG_INPUT_STABLE if input_stable else 0,
                                                _stream_handle()),
              "histogram256_u8")
    return bins


# ---- P: warp collectives --------------------------------------------------

def warp_collective(kind: str, a: torch.Tensor, b: torch.Tensor | None = None,
                    operand: int = 0, block: int = 32, width: int = 32,
                    mask: int = 0xFFFFFFFF, out: torch.Tensor | None = None) -> torch.Tensor:
    """Run one warp collective per logical thread (see include/warpfold_b200.h
    for the exact semantics).  ``a``: int32 operand per thread; ``b``: optional
    per-thread int32 offset / lane operand; threads outside ``mask`` leave
    ``out`` untouched."""
    if kind not in _lib.COLL:
        from .errors import UnsupportedFeatureError
        raise UnsupportedFeatureError(f"unknown warp collective {kind!r}")
    _require_cuda(a, torch.int32, "a")
    if b is not None:
        _require_cuda(b, torch.int32, "b")
        if b.numel() != a.numel():
            raise LaunchError("a and b must have the same length")
    if out is None:
        out = torch.zeros_like(a)
    _require_cuda(out, torch.int32, "out")
    with _on(a.device):
        check(_lib.load().wf_warp_collective(_lib.COLL[kind], a.data_ptr(),
                                             b.data_ptr() if b is not None else None,
                                             int(operand), out.data_ptr(), a.numel(), block, width,
                                             mask & 0xFFFFFFFF, _stream_handle()),
              "warp_collective")
    return out


# ---- synthetic inputs ------------------------------------------------------

_GEN_DTYPE = {"i32_full": torch.int32, "i32_small": torch.int32, "f32_unit": torch.float32,
              "u8_uniform": torch.uint8, "u8_const": torch.uint8, "u8_geom": torch.uint8,
              "i32_select": torch.int32}


def fill_synthetic(gen: str, n: int, seed: int = 0, base: int = 0, param: int = 0,
                   device=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Element i = f(splitmix64(seed ^ (base + i))) — identical to
    oracle/synthetic.py, generated directly in HBM."""
    if gen not in _lib.GEN:
        raise LaunchError(f"unknown generator {gen!r}")
    if out is None:
        device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        out = torch.empty(n, dtype=_GEN_DTYPE[gen], device=device)
    with _on(out.device):
        check(_lib.load().wf_fill_synthetic(_lib.GEN[gen], out.data_ptr(), n,
                                            seed & 0xFFFFFFFFFFFFFFFF, base, param,
                                            _stream_handle()),
              "fill_synthetic")
    return out


# ---- host-buffer (end-to-end) entry points --------------------------------

_staging_cache: dict = {}
STAGING_BYTES = 256 << 20


def _staging(device: torch.device) -> torch.Tensor:
    st = _staging_cache.get(device.index)
    if st is None:
        st = torch.empty(STAGING_BYTES, dtype=torch.uint8, device=device)
        _staging_cache[device.index] = st
    return st


def _host_ptr(arr) -> tuple[int, int]:
    if isinstance(arr, torch.Tensor):
        if arr.is_cuda or not arr.is_contiguous():
            raise LaunchError("host input must be a contiguous CPU tensor")
        return arr.data_ptr(), arr.numel()
    import numpy as np
    a = np.ascontiguousarray(arr)
    return a.ctypes.data, a.size


def reduce_sum_f32_host(host_x, device=None) -> float:
    """End-to-end fp32 sum of a host buffer (pinned for full PCIe speed):
    chunked H2D overlapped with K2, result copied back.  Synchronous."""
    import numpy as np
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    ptr, n = _host_ptr(host_x)
    out = np.zeros(1, dtype=np.float32)
    with _on(device):
        st = _staging(device)
        ws = workspace(_lib.OP_REDUCE_SUM_F32, n, device)
        check(_lib.load().wf_reduce_sum_f32_host(ptr, n, out.ctypes.data, st.data_ptr(), st.numel(),
                                                 ws.data_ptr(), ws.numel(), _stream_handle()),
              "reduce_sum_f32_host")
    return float(out[0])


def reduce_sum_i32_host(host_x, device=None) -> int:
    import numpy as np
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    ptr, n = _host_ptr(host_x)
    out = np.zeros(1, dtype=np.int32)
    with _on(device):
        st = _staging(device)
        ws = workspace(_lib.OP_REDUCE_SUM_I32, n, device)
        check(_lib.load().wf_reduce_sum_i32_host(ptr, n, out.ctypes.data, st.data_ptr(), st.numel(),
                                                 ws.data_ptr(), ws.numel(), _stream_handle()),
              "reduce_sum_i32_host")
    return int(out[0])


def histogram256_u8_host(host_x, device=None):
    import numpy as np
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    ptr, n = _host_ptr(host_x)
    out = np.zeros(256, dtype=np.uint64)
    with _on(device):
        st = _staging(device)
        ws = workspace(_lib.OP_HISTOGRAM256_U8, n, device)
        check(_lib.load().wf_histogram256_u8_host(ptr, n, out.ctypes.data, st.data_ptr(),
                                                  st.numel(), ws.data_ptr(), ws.numel(),
                                                  _stream_handle()),
              "histogram256_u8_host")
    return out


def _host_out(host_out, n: int, dtype):
    import numpy as np
    if host_out is None:
        return np.empty(n, dtype=dtype)
    if isinstance(host_out, torch.Tensor):
        if host_out.is_cuda or not host_out.is_contiguous() or host_out.numel() < n:
            raise LaunchError(f"host output must be a contiguous CPU tensor of >= {n} elements")
        return host_out
    a = host_out
    if not (isinstance(a, np.ndarray) and a.flags.c_contiguous and a.flags.writeable and
            a.dtype == dtype and a.size >= n):
        raise LaunchError(f"host output must be a writable contiguous {np.dtype(dtype)} array "
                          f"of >= {n} elements")
    return a


def _addr(a) -> int:
    return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data


def scan_inclusive_i32_host(host_x, host_out=None, carry: int | None = None, device=None):
    """End-to-end inclusive scan of a host buffer into a host buffer (pinned
    for full PCIe speed): H2D, K3 and D2H of successive chunks overlapped,
    one carry chain across chunks.  Synchronous; returns ``host_out``."""
    import ctypes
    import numpy as np
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    ptr, n = _host_ptr(host_x)
    out = _host_out(host_out, n, np.int32)
    cin = ctypes.c_int32(int(carry)) if carry is not None else None
    with _on(device):
        st = _staging(device)
        ws = workspace(_lib.OP_SCAN_INCLUSIVE_I32, STAGING_BYTES // 4, device)
        check(_lib.load().wf_scan_inclusive_i32_host(
            ptr, _addr(out), n, ctypes.addressof(cin) if cin is not None else None,
            st.data_ptr(), st.numel(), ws.data_ptr(), ws.numel(), _stream_handle()),
            "scan_inclusive_i32_host")
    return out


def compact_gt0_i32_host(host_x, host_out=None, device=None):
    """End-to-end order-preserving ``x[x > 0]`` from a host buffer into a host
    buffer.  Returns ``(host_out, count)``; the first ``count`` elements are
    the selected ones.  Synchronous."""
    import ctypes
    import numpy as np
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    ptr, n = _host_ptr(host_x)
    out = _host_out(host_out, n, np.int32)
    cnt = ctypes.c_uint64(0)
    with _on(device):
        st = _staging(device)
        ws = workspace(_lib.OP_COMPACT_GT0_I32, STAGING_BYTES // 4, device)
        check(_lib.load().wf_compact_gt0_i32_host(
            ptr, n, _addr(out), ctypes.addressof(cnt), st.data_ptr(), st.numel(),
            ws.data_ptr(), ws.numel(), _stream_handle()),
            "compact_gt0_i32_host")
    return out, int(cnt.value)
