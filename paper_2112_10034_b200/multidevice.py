"""Single-process multi-GPU: one host thread drives every device through the
``wf_mg_*`` C ABI (include/warpfold_b200.h; SURVEY.md §8b "wf_mg_init +
wf_mg_<op>").  Each call runs one kernel per rank with its exchange fused in
over peer memory — the same kernels the one-process-per-GPU path
(``p2p.PeerReducer`` / ``p2p.PeerCollectives``) uses — and returns once every
rank is done (the reference's join semantics, runtime/launch.py:1-8).

Reference anchor: the block-range split of one launch over workers
(runtime/launch.py:95-147, ``_split`` :137-147) applied across devices; the
caller passes each rank's contiguous shard (``split`` below is
``distributed.shard_range``).  Ranks may share a device (tests on one GPU).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib, ops
from .distributed import shard_range
from .errors import LaunchError


def _ptrs(ts, ctype=C.c_void_p):
    return (ctype * len(ts))(*[t.data_ptr() for t in ts])


class MultiDevice:
    """A ``wf_mg`` context over ``devices`` (one rank per entry)."""

    def __init__(self, devices):
        self.devices = [torch.device("cuda", int(d.index if isinstance(d, torch.device) else d))
                        for d in devices]
        arr = (C.c_int * len(self.devices))(*[d.index for d in self.devices])
        h = C.c_void_p()
        _lib.check(_lib.load().wf_mg_init(len(self.devices), arr, C.byref(h)), "wf_mg_init")
        self._h = h
        self._streams = []
        for r, d in enumerate(self.devices):
            s = C.c_void_p()
            _lib.check(_lib.load().wf_mg_stream(h, r, C.byref(s)), "wf_mg_stream")
            self._streams.append(torch.cuda.ExternalStream(s.value, device=d))

    @property
    def world(self) -> int:
        return len(self.devices)

    def split(self, x: torch.Tensor) -> list:
        """Contiguous shards of a host or device tensor, copied to the ranks'
        devices (the reference's ``_split`` on 4096-element granules)."""
        out = []
        for r, d in enumerate(self.devices):
            lo, hi = shard_range(x.numel(), r, self.world)
            out.append(x[lo:hi].to(d))
        return out

    # ---- plumbing -----------------------------------------------------------
    def _check_shards(self, shards, dtype, name):
        if len(shards) != self.world:
            raise LaunchError(f"{name}: {self.world} shards expected, got {len(shards)}")
        for s, d in zip(shards, self.devices):
            ops._require_cuda(s, dtype, name)
            if s.device != d:
                raise LaunchError(f"{name}: shard on {s.device}, rank device is {d}")

    def _call(self, fn, *args) -> None:
        # the ranks' streams start after the work already queued on each
        # device's current stream (the producers of the shards)
        for d, st in zip(self.devices, self._streams):
            st.wait_stream(torch.cuda.current_stream(d))
        lib = _lib.load()
        _lib.check(getattr(lib, fn)(self._h, *args), fn)
        _lib.check(lib.wf_mg_synchronize(self._h), "wf_mg_synchronize")

    # ---- ops ------------------------------------------------------------------
    def reduce_sum_f32(self, shards) -> list:
        """fp32 sum of all shards, bit-identical on every rank (one float32[1]
        per rank)."""
        self._check_shards(shards, torch.float32, "x")
        outs = [torch.empty(1, dtype=torch.float32, device=d) for d in self.devices]
        n = (C.c_uint64 * self.world)(*[s.numel() for s in shards])
        self._call("wf_mg_reduce_sum_f32", _ptrs(shards), n, _ptrs(outs))
        return outs

    def scan_inclusive_i32(self, shards, outs=None) -> list:
        """The global inclusive scan, each rank's part on its device."""
        self._check_shards(shards, torch.int32, "x")
        outs = outs if outs is not None else [torch.empty_like(s) for s in shards]
        n = (C.c_uint64 * self.world)(*[s.numel() for s in shards])
        self._call("wf_mg_scan_inclusive_i32", _ptrs(shards), _ptrs(outs), n)
        return outs

    def compact_gt0_i32(self, shards, outs=None):
        """(outs, counts3): rank r's selected elements in outs[r][:count] and
        counts3[r] = int64[3] {count, global offset, global total}; the
        concatenation over ranks is ``x[x > 0]``."""
        self._check_shards(shards, torch.int32, "x")
        outs = outs if outs is not None else [torch.empty_like(s) for s in shards]
        c3 = [torch.empty(3, dtype=torch.int64, device=d) for d in self.devices]
        n = (C.c_uint64 * self.world)(*[s.numel() for s in shards])
        self._call("wf_mg_compact_gt0_i32", _ptrs(shards), n, _ptrs(outs), _ptrs(c3))
        return outs, c3

    def histogram256_u8(self, shards) -> list:
        """The global 256 bins (int64) on every rank."""
        self._check_shards(shards, torch.uint8, "x")
        bins = [torch.empty(256, dtype=torch.int64, device=d) for d in self.devices]
        n = (C.c_uint64 * self.world)(*[s.numel() for s in shards])
        self._call("wf_mg_histogram256_u8", _ptrs(shards), n, _ptrs(bins))
        return bins

    def close(self) -> None:
        if self._h:
            _lib.load().wf_mg_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
