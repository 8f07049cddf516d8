"""Multi-GPU sharding of the warp-primitive path: one process per GPU,
``torch.distributed`` over NCCL (NVLink 5 / NVSwitch) for the exchanges.

The reference's only parallelism is block-range data parallelism over CPU
workers (runtime/launch.py:95-128, ``_split`` at :137-147).  Here the same
contiguous-range split is applied across GPUs; every shard is
processed by the single-GPU kernel and the per-GPU partials are combined by
one small collective:

  reduce_sum_f32 / _i32  all-gather of one partial per rank, then the same
                         fixed-order fold kernel on every rank (deterministic,
                         bit-identical on all ranks; no fp atomics)
  scan_inclusive_i32     reduce -> all-gather of shard totals -> exclusive
                         carry (fold of the first `rank` totals, on device) ->
                         scan with carry-in (12 B/elem instead of 8)
  compact_gt0_i32        local ordered compaction -> all-gather of counts ->
                         global offset (output stays sharded; the
                         concatenation over ranks is a[a > 0])
  histogram256_u8        local bins -> all-reduce(sum) of 256 counters

The exchange helpers are backend-agnostic (NCCL on GPUs, gloo in the CPU
tests) and the carries/offsets are computed by the device kernels, so a step
needs no host round trip.  With a ``p2p.PeerCollectives`` (``peer=``) the
exchanges travel over peer memory (NVLink, CUDA IPC mailboxes) instead, each
inside the kernel that produces its input (scan pass 1, compaction,
histogram: one kernel per rank and op); the fp32 reduction has its own fused
form (``p2p.PeerReducer``).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import ops

GRANULE = 4096  # shard boundaries on 16 KiB (int32) / 4 KiB (u8) multiples


def shard_range(n: int, rank: int, world: int, granule: int = GRANULE) -> tuple[int, int]:
    """Contiguous shard of [0, n) for ``rank`` — the reference's ``_split``
    (runtime/launch.py:137-147) applied to granules instead of blocks, so
    every shard starts 16-byte aligned."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    units = (n + granule - 1) // granule
    base, extra = divmod(units, world)
    lo_u = rank * base + min(rank, extra)
    hi_u = lo_u + base + (1 if rank < extra else 0)
    return min(n, lo_u * granule), min(n, hi_u * granule)


def _world(group=None) -> tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def exchange(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather of a small per-rank tensor -> [world, *local.shape]."""
    rank, world = _world(group)
    if world == 1:
        return local.reshape(1, *local.shape)
    flat = local.contiguous().reshape(-1)
    out = torch.empty(world * flat.numel(), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, flat, group=group)
    return out.reshape(world, *local.shape)


def reduce_sum_f32(x_local: torch.Tensor, group=None, block: int = 256) -> torch.Tensor:
    part = ops.reduce_sum_f32(x_local, block=block)
    rank, world = _world(group)
    if world == 1:
        return part
    return ops.fold(exchange(part, group).reshape(-1))


def reduce_sum_i32(x_local: torch.Tensor, group=None, block: int = 256) -> torch.Tensor:
    part = ops.reduce_sum_i32(x_local, block=block)
    rank, world = _world(group)
    if world == 1:
        return part
    return ops.fold(exchange(part, group).reshape(-1))


def cyclic_rounds(n: int, rank: int, world: int, round_elems: int = 1 << 22):
    """Block-cyclic layout of a global array of `n` elements: global
    super-tile g (`round_elems` elements, the last one short) lives on rank
    g % world.  Returns (rounds, [(global_start, length), ...] of this
    rank's super-tiles in local order); `rounds` is the same on every rank
    (ranks with fewer super-tiles contribute empty rounds)."""
    supers = -(-n // round_elems)
    rounds = -(-supers // world)
    mine = []
    for r in range(rounds):
        g = r * world + rank
        if g < supers:
            start = g * round_elems
            mine.append((start, min(round_elems, n - start)))
    return rounds, mine


def scan_inclusive_i32(x_local: torch.Tensor, out: torch.Tensor | None = None,
                       group=None, peer=None, input_stable: bool = False) -> torch.Tensor:
    """`peer`: a p2p.PeerCollectives — the shard totals then travel over peer
    memory in one kernel instead of NCCL all-gather + fold.  `input_stable`:
    WF_FLAG_INPUT_STABLE for the first kernel of the call (the kernel issued
    just before on the stream does not write `x_local`); the scan after the
    fused pass 1 always takes it (pass 1 writes only the carry)."""
    rank, world = _world(group)
    if world == 1:
        return ops.scan_inclusive_i32(x_local, out, input_stable=input_stable)
    if peer is not None:  # pass 1 + carry exchange in one kernel
        carry = peer.reduce_exscan_i32(x_local, input_stable=input_stable)[:1]
        return ops.scan_inclusive_i32(x_local, out, carry=carry, input_stable=True)
    totals = exchange(ops.reduce_sum_i32(x_local), group).reshape(-1)
    carry = ops.fold(totals, count=rank)  # exclusive prefix of earlier shards
    return ops.scan_inclusive_i32(x_local, out, carry=carry)


def compact_gt0_i32(x_local: torch.Tensor, out: torch.Tensor | None = None, group=None,
                    peer=None, input_stable: bool = False):
    """Returns (out_local, count_local, offset, total) as device int64 scalars
    for count/offset/total; rank r's selected elements belong at
    [offset, offset + count) of the global a[a > 0].  `input_stable`:
    WF_FLAG_INPUT_STABLE."""
    rank, world = _world(group)
    if world > 1 and peer is not None:  # compaction + offset exchange in one kernel
        out, c3 = peer.compact_gt0_i32(x_local, out, input_stable=input_stable)
        return out, c3[:1], c3[1:2], c3[2:]
    out, count = ops.compact_gt0_i32(x_local, out, input_stable=input_stable)
    if world == 1:
        zero = torch.zeros(1, dtype=torch.int64, device=count.device)
        return out, count, zero, count
    counts = exchange(count, group).reshape(-1)
    offset = ops.fold(counts, count=rank)
    total = ops.fold(counts)
    return out, count, offset, total


def histogram256_u8(x_local: torch.Tensor, group=None, peer=None,
                    input_stable: bool = False) -> torch.Tensor:
    """`input_stable`: WF_FLAG_INPUT_STABLE (the kernel issued just before on
    the stream does not write `x_local`)."""
    rank, world = _world(group)
    if world > 1 and peer is not None:  # histogram + bin all-reduce in one kernel
        return peer.histogram256_u8(x_local, input_stable=input_stable)
    bins = ops.histogram256_u8(x_local, input_stable=input_stable)
    if world > 1:
        dist.all_reduce(bins, op=dist.ReduceOp.SUM, group=group)
    return bins
