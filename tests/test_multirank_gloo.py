"""N>1 host logic on CPU: world_size-2 gloo process group.

The per-shard compute here is the oracle (test-only stand-in for the sm_100a
kernel); what is under test is the product's sharding (distributed.shard_range,
the reference's _split applied to granules) and exchange (distributed.exchange,
the all-gather every sharded op uses), plus the combine rules of SURVEY.md
§8e: fixed-order fold of partials, exclusive carries for the scan, global
offsets for the compaction, and the bin all-reduce for the histogram."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import numpy_oracle as no, synthetic
from paper_2112_10034_b200 import distributed as wd


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = wd.shard_range(n, rank, world)
        res = {}
        # C2: per-rank fp32 partial -> all-gather -> fixed-order fold (same bits on all ranks)
        f = synthetic.generate("f32_unit", hi - lo, seed=1, base=lo)
        part = torch.tensor([float(np.float32(no.reduce_sum_f32_exact(f)))], dtype=torch.float32)
        g = wd.exchange(part).reshape(-1).numpy()
        res["f32_parts"] = g.tolist()
        # C1-style wrapping i32 partials
        a = synthetic.generate("i32_full", hi - lo, seed=2, base=lo)
        ip = torch.tensor([no.reduce_sum_i32(a)], dtype=torch.int32)
        res["i32_total"] = no.reduce_sum_i32(wd.exchange(ip).reshape(-1).numpy())
        # C3: totals -> exclusive carry -> local scan with carry
        totals = wd.exchange(ip).reshape(-1).numpy()
        carry = no.reduce_sum_i32(totals[:rank]) if rank else 0
        res["scan"] = no.scan_inclusive_i32(a, carry=carry)
        # C4: counts -> global offset; output stays sharded
        sel = no.compact_gt0_i32(a)
        counts = wd.exchange(torch.tensor([len(sel)], dtype=torch.int64)).reshape(-1).numpy()
        res["compact"] = (int(counts[:rank].sum()), sel, int(counts.sum()))
        # C5: bins all-reduce
        u = synthetic.generate("u8_uniform", hi - lo, seed=3, base=lo)
        bins = torch.from_numpy(no.histogram256_u8(u).astype(np.int64))
        dist.all_reduce(bins, op=dist.ReduceOp.SUM)
        res["bins"] = bins.numpy()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_and_combine():
    world, n = 2, 100_003
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank saw the same gathered partials (rank order)
    assert out[0]["f32_parts"] == out[1]["f32_parts"]
    f = synthetic.generate("f32_unit", n, seed=1)
    assert abs(sum(out[0]["f32_parts"]) - no.reduce_sum_f32_exact(f)) <= \
        no.f32_tolerance(n, no.abs_sum(f))
    a = synthetic.generate("i32_full", n, seed=2)
    assert out[0]["i32_total"] == out[1]["i32_total"] == no.reduce_sum_i32(a)
    assert np.array_equal(np.concatenate([out[0]["scan"], out[1]["scan"]]),
                          no.scan_inclusive_i32(a))
    off0, sel0, tot = out[0]["compact"]
    off1, sel1, _ = out[1]["compact"]
    assert off0 == 0 and off1 == len(sel0)
    glob = np.empty(tot, dtype=np.int32)
    glob[off0:off0 + len(sel0)] = sel0
    glob[off1:off1 + len(sel1)] = sel1
    assert np.array_equal(glob, no.compact_gt0_i32(a))
    u = synthetic.generate("u8_uniform", n, seed=3)
    assert np.array_equal(out[0]["bins"].astype(np.uint64), no.histogram256_u8(u))
    assert np.array_equal(out[1]["bins"], out[0]["bins"])


@pytest.mark.parametrize("n,world", [(0, 1), (1, 2), (4096, 2), (4097, 2), (10**6, 8),
                                     (1 << 30, 8), (1 << 32, 3), (12345, 7)])
def test_shard_range_partitions(n, world):
    ranges = [wd.shard_range(n, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    for lo, _ in ranges:
        assert lo % wd.GRANULE == 0 or lo == n  # 16-byte aligned shard starts
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 2 * wd.GRANULE


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        wd.shard_range(10, 2, 2)


def _p2p_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2112_10034_b200 import p2p
        try:
            p2p.Mailboxes.from_process_group(torch.device("cpu"))
            q.put((rank, "built"))
        except Exception as e:  # expected here: no GPU for the mailbox
            q.put((rank, f"raised {type(e).__name__}"))
        dist.barrier()  # every rank left the set-up collective sequence together
    finally:
        dist.destroy_process_group()


def test_peer_mailbox_setup_failure_is_collective():
    """Without a GPU the mailbox allocation fails; the set-up is a consensus
    collective, so EVERY rank raises (and none is left waiting in a
    collective) — the bench then keeps the NCCL exchange on all ranks."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out == {0: "raised LaunchError", 1: "raised LaunchError"}


def _cyclic_worker(rank, world, port, n, round_elems, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rounds, parts = wd.cyclic_rounds(n, rank, world, round_elems)
        full = synthetic.generate("i32_full", n, seed=8)
        local = [full[s:s + m] for s, m in parts]
        # every rank's total of every round (0 for rounds it has no data in):
        # what the kernel's totaler publishes into the peer mailboxes
        mine = np.zeros(rounds, dtype=np.int64)
        for r, a in enumerate(local):
            mine[r] = no.reduce_sum_i32(a) & 0xFFFFFFFF
        totals = wd.exchange(torch.from_numpy(mine)).reshape(world, rounds).numpy()
        # the sweeper's rule: round r starts at (all ranks' earlier rounds)
        # + (lower ranks' round r)
        out, before = [], 0
        for r, a in enumerate(local):
            start = (before + int(totals[:rank, r].sum())) & 0xFFFFFFFF
            out.append((parts[r][0], no.scan_inclusive_i32(a, carry=np.int32(np.uint32(start)))))
            before = (before + int(totals[:, r].sum())) & 0xFFFFFFFF
        q.put((rank, rounds, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 5 * 4096 + 77), (3, 11 * 4096), (2, 4096)])
def test_cyclic_scan_combine_rule_two_ranks(world, n):
    """The block-cyclic sharded scan's host layout (distributed.cyclic_rounds)
    and the per-round combine rule its kernel implements, over a real gloo
    process group: stitched back in global order the ranks' super-tiles equal
    the global inclusive scan.  Every rank sees the same round count."""
    round_elems = 4096
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cyclic_worker, args=(r, world, port, n, round_elems, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len({rounds for _, rounds, _ in got}) == 1
    pieces = sorted((start, arr) for _, _, out in got for start, arr in out)
    stitched = np.concatenate([arr for _, arr in pieces])
    assert [s for s, _ in pieces] == list(range(0, n, round_elems))
    full = synthetic.generate("i32_full", n, seed=8)
    assert np.array_equal(stitched, no.scan_inclusive_i32(full))

