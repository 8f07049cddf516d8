"""Fused reduce + exchange over peer memory (NVLink 5 / NVSwitch) for the
sharded fp32 reduction (BASELINE config 2).

The NCCL path of ``distributed.reduce_sum_f32`` is three stream operations per
step: the K2 kernel, an all-gather of one float per rank and the fixed-order
fold kernel.  ``PeerReducer`` makes it ONE kernel per rank
(``wf_reduce_sum_f32_mg``): the kernel's last block stores the rank partial
straight into every rank's mailbox through CUDA IPC mappings and folds the
arriving partials with the same association as ``wf_fold_f32`` — so the result
is bit-identical to the NCCL path and on every rank.  Mailbox handles are
exchanged once, at construction, through ``torch.distributed``.

Reference anchor: the reference's only parallelism is the block-range split
over CPU workers with join semantics (runtime/launch.py:95-147); SURVEY.md §8e
maps C2 to "independent units + one exchange".
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _lib, ops
from .errors import LaunchError


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise LaunchError(f"{what}: {_lib.last_error()}")


class Mailboxes:
    """`world` mailboxes and the device array of their pointers, as seen by
    one rank.  Built either across processes (``from_process_group``) or
    inside one process for tests (``local``: all mailboxes on this device)."""

    def __init__(self, own: int, ptrs: list[int], opened: list[int], device: torch.device,
                 owned: list[int]):
        self.own = own
        self.ptrs = ptrs
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=device)
        self._opened = opened
        self._owned = owned

    @staticmethod
    def _alloc(world: int, cap: int | None, out: C.c_void_p) -> None:
        lib = _lib.load()
        if cap is None:  # the fused-K2 layout: one epoch-tagged word per rank and bank
            _check(lib.wf_mailbox_alloc(world, C.byref(out)), "wf_mailbox_alloc")
        else:            # wf_peer_exchange layout: `cap` payload words + flag per rank and bank
            _check(lib.wf_peer_mailbox_alloc(world, cap, C.byref(out)), "wf_peer_mailbox_alloc")

    @classmethod
    def from_process_group(cls, device: torch.device, group=None,
                           cap: int | None = None) -> "Mailboxes":
        """Collective: every rank of `group` must call it.  Failures on any
        rank (no IPC, no peer access) make every rank raise, after the same
        sequence of collectives, so no rank is left waiting in one."""
        lib = _lib.load()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        mine, handle, err = C.c_void_p(), (C.c_char * 64)(), None
        try:
            cls._alloc(world, cap, mine)
            _check(lib.wf_ipc_handle(mine, handle), "wf_ipc_handle")
        except LaunchError as e:
            err = str(e)
        handles: list = [None] * world
        dist.all_gather_object(handles, None if err else bytes(handle), group=group)
        ptrs, opened = [], []
        if err is None:
            try:
                for r, h in enumerate(handles):
                    if r == rank:
                        ptrs.append(mine.value)
                        continue
                    if h is None:
                        raise LaunchError(f"rank {r} could not export its mailbox")
                    p = C.c_void_p()
                    _check(lib.wf_ipc_open(C.create_string_buffer(h, 64), C.byref(p)), "wf_ipc_open")
                    ptrs.append(p.value)
                    opened.append(p.value)
            except LaunchError as e:
                err = str(e)
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        box = cls(mine.value, ptrs if not err else [0] * world, opened, device,
                  [mine.value] if mine.value else [])
        if int(ok.item()) != 1:
            box.close()
            raise LaunchError(err or "a peer rank could not set up its mailbox")
        return box

    @classmethod
    def local(cls, world: int, device: torch.device, cap: int | None = None) -> list["Mailboxes"]:
        """In-process stand-in for `world` ranks on one GPU (tests): every
        rank's view shares the same pointer array."""
        own = []
        for _ in range(world):
            p = C.c_void_p()
            cls._alloc(world, cap, p)
            own.append(p.value)
        views = [cls(own[r], own, [], device, []) for r in range(world)]
        views[0]._owned = own  # freed once
        return views

    def close(self) -> None:
        lib = _lib.load()
        for p in self._opened:
            lib.wf_ipc_close(C.c_void_p(p))
        for p in self._owned:
            lib.wf_mailbox_free(C.c_void_p(p))
        self._opened, self._owned = [], []


class PeerReducer:
    """`reduce_sum_f32` of the sharded input, exchanged over peer memory."""

    def __init__(self, boxes: Mailboxes, rank: int, world: int):
        self.boxes, self.rank, self.world = boxes, rank, world
        self.epoch = 0

    @classmethod
    def for_process_group(cls, device: torch.device, group=None) -> "PeerReducer":
        boxes = Mailboxes.from_process_group(device, group)
        return cls(boxes, dist.get_rank(group), dist.get_world_size(group))

    def reduce_sum_f32(self, x_local: torch.Tensor, out: torch.Tensor | None = None,
                       block: int = 256, stream=None, input_stable: bool = False) -> torch.Tensor:
        """``input_stable``: as ``ops.reduce_sum_f32`` (WF_FLAG_INPUT_STABLE)."""
        ops._require_cuda(x_local, torch.float32, "x")
        if out is None:
            out = torch.empty(1, dtype=torch.float32, device=x_local.device)
        self.epoch += 1
        ws = ops.workspace(_lib.OP_REDUCE_SUM_F32, x_local.numel(), x_local.device, stream)
        lib = _lib.load()
        _check(lib.wf_reduce_sum_f32_mg_ex(x_local.data_ptr(), x_local.numel(), out.data_ptr(),
                                           block, 0, ws.data_ptr(), ws.numel(),
                                           self.boxes.peers.data_ptr(), self.boxes.own,
                                           self.rank, self.world, self.epoch,
                                           _lib.FLAG_INPUT_STABLE if input_stable else 0,
                                           ops._stream_handle(stream)),
               "wf_reduce_sum_f32_mg")
        return out

    def close(self) -> None:
        self.boxes.close()


class PeerCollectives:
    """The exchanges of the sharded C3-C5 paths over peer memory, results
    identical on every rank, each fused into the kernel that produces its
    input (`reduce_exscan_i32`: scan pass 1 + carry; `compact_gt0_i32`:
    compaction + offsets; `histogram256_u8`: bins + all-reduce); the
    stand-alone single-block exchanges (`exscan_u32`, `exscan_u64`,
    `allreduce_u64`) serve any other value.  All share one mailbox and epoch
    sequence; every rank must issue the same sequence of calls."""

    EXSCAN, ALLREDUCE, EXSCAN_U32 = 1, 2, 3

    def __init__(self, boxes: Mailboxes, rank: int, world: int, cap: int, device: torch.device):
        self.boxes, self.rank, self.world, self.cap = boxes, rank, world, cap
        self.epoch = 0
        self.err = torch.zeros(1, dtype=torch.int32, device=device)

    @classmethod
    def for_process_group(cls, device: torch.device, group=None, cap: int = 256):
        boxes = Mailboxes.from_process_group(device, group, cap=cap)
        return cls(boxes, dist.get_rank(group), dist.get_world_size(group), cap, device)

    def _run(self, mode: int, vals: torch.Tensor, count: int, out: torch.Tensor, stream=None):
        self.epoch += 1
        _check(_lib.load().wf_peer_exchange(mode, vals.data_ptr(), count, self.cap, out.data_ptr(),
                                            self.boxes.peers.data_ptr(), self.boxes.own,
                                            self.rank, self.world, self.epoch,
                                            self.err.data_ptr(), ops._stream_handle(stream)),
               "wf_peer_exchange")
        return out

    def exscan_u32(self, v: torch.Tensor, stream=None) -> torch.Tensor:
        """int32[1] per rank -> int32[2] = (sum over lower ranks, sum over all), mod 2^32."""
        out = torch.empty(2, dtype=torch.int32, device=v.device)
        return self._run(self.EXSCAN_U32, v, 1, out, stream)

    def exscan_u64(self, v: torch.Tensor, stream=None) -> torch.Tensor:
        """int64[1] per rank -> int64[2] = (sum over lower ranks, sum over all)."""
        out = torch.empty(2, dtype=torch.int64, device=v.device)
        return self._run(self.EXSCAN, v, 1, out, stream)

    def allreduce_u64(self, v: torch.Tensor, stream=None) -> torch.Tensor:
        """int64[count] per rank -> elementwise sum over ranks (wrapping)."""
        out = torch.empty_like(v)
        return self._run(self.ALLREDUCE, v, v.numel(), out, stream)

    def reduce_exscan_i32(self, x_local: torch.Tensor, out: torch.Tensor | None = None,
                          block: int = 256, stream=None, input_stable: bool = False) -> torch.Tensor:
        """K1 over this rank's shard with the carry exchange fused into its
        last block (``wf_reduce_sum_i32_exscan_mg``): int32[2] = (wrapping sum
        of the shards of lower ranks, wrapping sum of all shards) — the
        sharded scan's pass 1 + exchange in one kernel."""
        ops._require_cuda(x_local, torch.int32, "x")
        if out is None:
            out = torch.empty(2, dtype=torch.int32, device=x_local.device)
        self.epoch += 1
        ws = ops.workspace(_lib.OP_REDUCE_SUM_I32, x_local.numel(), x_local.device, stream)
        _check(_lib.load().wf_reduce_sum_i32_exscan_mg_ex(
            x_local.data_ptr(), x_local.numel(), out.data_ptr(), block, 0, ws.data_ptr(),
            ws.numel(), self.boxes.peers.data_ptr(), self.boxes.own, self.cap, self.rank,
            self.world, self.epoch, self.err.data_ptr(),
            _lib.FLAG_INPUT_STABLE if input_stable else 0, ops._stream_handle(stream)),
            "wf_reduce_sum_i32_exscan_mg")
        return out

    def scan_inclusive_i32_cyclic(self, x_local: torch.Tensor, out: torch.Tensor | None = None,
                                  round_elems: int = 1 << 22, rounds: int | None = None,
                                  max_grid: int = 0, stream=None,
                                  input_stable: bool = False) -> torch.Tensor:
        """Single-pass scan of a BLOCK-CYCLIC sharded array
        (``wf_scan_inclusive_i32_cyclic_mg``): global super-tile g of
        `round_elems` elements lives on rank g % world; `x_local` holds this
        rank's super-tiles back to back (``distributed.cyclic_rounds``) and
        `out` receives the global inclusive scan at those positions.  The
        round totals are all-gathered inside the scan kernel, so each element
        is read once (8 B/elem).  `rounds`: the same on every rank (default:
        this rank's own count — pass the global count when shards differ)."""
        ops._require_cuda(x_local, torch.int32, "x")
        if out is None:
            out = torch.empty_like(x_local)
        if rounds is None:
            rounds = -(-x_local.numel() // round_elems)
        self.epoch += 1
        ws = ops.workspace(_lib.OP_SCAN_INCLUSIVE_I32, x_local.numel(), x_local.device, stream)
        _check(_lib.load().wf_scan_inclusive_i32_cyclic_mg(
            x_local.data_ptr(), out.data_ptr(), x_local.numel(), ws.data_ptr(), ws.numel(),
            self.boxes.peers.data_ptr(), self.boxes.own, self.cap, self.rank, self.world,
            self.epoch, self.err.data_ptr(), round_elems, rounds, max_grid,
            _lib.FLAG_INPUT_STABLE if input_stable else 0, ops._stream_handle(stream)),
            "wf_scan_inclusive_i32_cyclic_mg")
        return out

    def compact_gt0_i32(self, x_local: torch.Tensor, out: torch.Tensor | None = None,
                        stream=None, input_stable: bool = False):
        """K4 over this rank's shard with the offset exchange fused into the
        compaction kernel (``wf_compact_gt0_i32_mg``): returns (out_local,
        int64[3] = (count, global offset, global total))."""
        ops._require_cuda(x_local, torch.int32, "x")
        if out is None:
            out = torch.empty_like(x_local)
        counts = torch.empty(3, dtype=torch.int64, device=x_local.device)
        self.epoch += 1
        ws = ops.workspace(_lib.OP_COMPACT_GT0_I32, x_local.numel(), x_local.device, stream)
        _check(_lib.load().wf_compact_gt0_i32_mg_ex(
            x_local.data_ptr(), x_local.numel(), out.data_ptr(), counts.data_ptr(), ws.data_ptr(),
            ws.numel(), self.boxes.peers.data_ptr(), self.boxes.own, self.cap, self.rank,
            self.world, self.epoch, self.err.data_ptr(),
            _lib.FLAG_INPUT_STABLE if input_stable else 0, ops._stream_handle(stream)),
            "wf_compact_gt0_i32_mg")
        return out, counts

    def histogram256_u8(self, x_local: torch.Tensor, bins: torch.Tensor | None = None,
                        stream=None, input_stable: bool = False) -> torch.Tensor:
        """K5 over this rank's shard with the bin all-reduce fused into its
        last block (``wf_histogram256_u8_mg``): the global int64[256] bins on
        every rank.  ``input_stable``: WF_FLAG_INPUT_STABLE."""
        ops._require_cuda(x_local, torch.uint8, "x")
        if bins is None:
            bins = torch.empty(256, dtype=torch.int64, device=x_local.device)
        self.epoch += 1
        ws = ops.workspace(_lib.OP_HISTOGRAM256_U8, x_local.numel(), x_local.device, stream)
        _check(_lib.load().wf_histogram256_u8_mg_ex(
            x_local.data_ptr(), x_local.numel(), bins.data_ptr(), ws.data_ptr(), ws.numel(),
            self.boxes.peers.data_ptr(), self.boxes.own, self.cap, self.rank, self.world,
            self.epoch, self.err.data_ptr(), _lib.FLAG_INPUT_STABLE if input_stable else 0,
            ops._stream_handle(stream)),
            "wf_histogram256_u8_mg")
        return bins

    def failed(self) -> bool:
        """True once any call timed out waiting for a peer (~4 s); sticky
        until clear_error().  Synchronises with the device."""
        return bool(self.err.item())

    def clear_error(self) -> None:
        self.err.zero_()

    def close(self) -> None:
        self.boxes.close()


def try_peer_reducer(device: torch.device, x_probe: torch.Tensor, group=None):
    """Collective.  Build a PeerReducer and check it bit-for-bit against the
    NCCL path on `x_probe` (this rank's shard of a probe input).  Returns
    (reducer, "ok") or (None, reason) — the same outcome on every rank."""
    from . import distributed as wd
    try:
        pr = PeerReducer.for_process_group(device, group)
    except Exception as e:  # identical on all ranks (consensus inside)
        return None, f"{type(e).__name__}: {e}"
    want = wd.reduce_sum_f32(x_probe, group=group)
    got = pr.reduce_sum_f32(x_probe)
    same = torch.equal(got.view(torch.int32), want.view(torch.int32))
    ok = torch.tensor([1 if same else 0], dtype=torch.int32, device=device)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if int(ok.item()) != 1:
        pr.close()
        return None, "peer-memory result differs from the NCCL path"
    return pr, "ok"


def try_peer_collectives(device: torch.device, group=None, cap: int = 256):
    """Collective.  PeerCollectives checked against NCCL on a probe (an
    exclusive scan of rank+1, an all-reduce of a rank-dependent vector, and
    the two fused kernels: scan pass 1 + carry, histogram + bin all-reduce).
    Returns (collectives, "ok") or (None, reason) — the same on every rank."""
    from . import distributed as wd
    try:
        pc = PeerCollectives.for_process_group(device, group, cap)
    except Exception as e:
        return None, f"{type(e).__name__}: {e}"
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    v = torch.tensor([rank + 1], dtype=torch.int64, device=device)
    got = pc.exscan_u64(v)
    vec = torch.arange(cap, dtype=torch.int64, device=device) * (rank + 3)
    red = pc.allreduce_u64(vec)
    gathered = wd.exchange(v, group).reshape(-1)
    want_red = vec.clone()
    dist.all_reduce(want_red, group=group)
    xi = ops.fill_synthetic("i32_full", 100003 + 17 * rank, seed=rank, device=device)
    carry = pc.reduce_exscan_i32(xi)
    totals = wd.exchange(ops.reduce_sum_i32(xi), group).reshape(-1).to(torch.int64) & 0xFFFFFFFF
    xu = ops.fill_synthetic("u8_uniform", 300007 + 5 * rank, seed=rank, device=device)
    bins = pc.histogram256_u8(xu)
    want_bins = ops.histogram256_u8(xu)
    dist.all_reduce(want_bins, group=group)
    _, cnt3 = pc.compact_gt0_i32(xi)
    counts = wd.exchange(ops.compact_gt0_i32(xi)[1], group).reshape(-1)
    same = (not pc.failed() and int(got[0]) == int(gathered[:rank].sum())
            and int(got[1]) == int(gathered.sum()) and torch.equal(red, want_red)
            and int(carry[0]) & 0xFFFFFFFF == int(totals[:rank].sum()) & 0xFFFFFFFF
            and int(carry[1]) & 0xFFFFFFFF == int(totals.sum()) & 0xFFFFFFFF
            and torch.equal(bins, want_bins)
            and cnt3.tolist() == [int(counts[rank]), int(counts[:rank].sum()), int(counts.sum())])
    ok = torch.tensor([1 if same else 0], dtype=torch.int32, device=device)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if int(ok.item()) != 1:
        pc.close()
        return None, "peer-memory collectives differ from NCCL"
    return pc, "ok"
