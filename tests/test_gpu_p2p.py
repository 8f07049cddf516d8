"""Fused reduce + exchange over peer memory (wf_reduce_sum_f32_mg,
paper_2112_10034_b200/p2p.py).

Multi-GPU boxes are not available to these tests, so the protocol runs with
`world` ranks inside one process on one GPU: every rank's kernel on its own
stream, all mailboxes in this device's memory.  The kernels really run
concurrently and really wait for each other, so epochs, bank alternation,
late ranks and the fold association are exercised; the result must be
bit-identical on every rank and to the NCCL path (per-rank K2 partials ->
all-gather -> wf_fold_f32).  A second test maps a mailbox into another
process through the CUDA IPC handle path the multi-process code uses."""

import multiprocessing as mp

import numpy as np

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import numpy_oracle as no, synthetic  # noqa: E402


@pytest.fixture(scope="module")
def mods():
    from paper_2112_10034_b200 import build
    build.build_library()
    from paper_2112_10034_b200 import distributed, ops, p2p
    torch.cuda.init()
    return ops, p2p, distributed


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_fused_exchange_in_process(mods, world):
    ops, p2p, wd = mods
    dev = torch.device("cuda", 0)
    n = (1 << 22) * world + 1234
    shards = [wd.shard_range(n, r, world) for r in range(world)]
    xs = [ops.fill_synthetic("f32_unit", hi - lo, seed=9, base=lo) for lo, hi in shards]
    want = ops.fold(torch.cat([ops.reduce_sum_f32(x) for x in xs]))  # the NCCL path's combine
    whole = synthetic.generate("f32_unit", n, seed=9)
    assert abs(float(want.item()) - no.reduce_sum_f32_exact(whole)) <= no.f32_tolerance(n, no.abs_sum(whole))
    boxes = p2p.Mailboxes.local(world, dev)
    reducers = [p2p.PeerReducer(boxes[r], r, world) for r in range(world)]
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    torch.cuda.synchronize()
    try:
        for step in range(5):
            order = range(world) if step % 2 == 0 else reversed(range(world))
            outs = [None] * world
            for r in order:  # odd steps launch the last rank first
                with torch.cuda.stream(streams[r]):
                    outs[r] = reducers[r].reduce_sum_f32(xs[r], stream=streams[r])
            torch.cuda.synchronize()
            for r in range(world):
                assert torch.equal(outs[r].view(torch.int32), want.view(torch.int32)), (step, r)
    finally:
        torch.cuda.synchronize()
        boxes[0].close()


def test_fused_exchange_input_stable_chain(mods):
    """wf_reduce_sum_f32_mg_ex with WF_FLAG_INPUT_STABLE (what bench.py's
    headline steps use at N>1): a back-to-back chain of dependent launches on
    one mailbox, epochs alternating banks, every result bit-identical to the
    plain fused launch (world 1: own mailbox only; ranks sharing one GPU are
    not chained, they would compete for SM slots with their own successors)."""
    ops, p2p, wd = mods
    dev = torch.device("cuda", 0)
    x = ops.fill_synthetic("f32_unit", (1 << 23) + 77, seed=3)
    boxes = p2p.Mailboxes.local(1, dev)
    try:
        pr = p2p.PeerReducer(boxes[0], 0, 1)
        want = pr.reduce_sum_f32(x).clone()
        torch.cuda.synchronize()
        outs = torch.empty(12, dtype=torch.float32, device=dev)
        for k in range(12):
            pr.reduce_sum_f32(x, outs[k:k + 1], input_stable=True)
        torch.cuda.synchronize()
        assert torch.equal(outs.view(torch.int32), want.view(torch.int32).expand(12))
    finally:
        torch.cuda.synchronize()
        boxes[0].close()


def test_fused_histogram_input_stable_chain(mods):
    """wf_histogram256_u8_mg_ex with WF_FLAG_INPUT_STABLE, world 1: a chain of
    dependent launches on one mailbox, every result equal to the plain one."""
    ops, p2p, wd = mods
    dev = torch.device("cuda", 0)
    u = ops.fill_synthetic("u8_geom", (1 << 24) + 3, seed=2)
    boxes = p2p.Mailboxes.local(1, dev, cap=256)
    try:
        pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)
        want = pc.histogram256_u8(u).clone()
        torch.cuda.synchronize()
        bins = torch.empty(8, 256, dtype=torch.int64, device=dev)
        for k in range(8):
            pc.histogram256_u8(u, bins[k], input_stable=True)
        torch.cuda.synchronize()
        assert torch.equal(bins, want.expand(8, 256)) and not pc.failed()
    finally:
        torch.cuda.synchronize()
        boxes[0].close()


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_cyclic_scan_in_process(mods, world):
    """Single-pass scan of a block-cyclic sharded array, every rank a
    concurrent kernel on its own stream of the one GPU (grids capped so all
    ranks are resident at once: the rounds wait on each other mid-kernel).
    Each rank's output equals the global inclusive scan at its positions;
    three calls in a row (epoch banks alternate), plain and dependent
    launches."""
    ops, p2p, wd = mods
    dev = torch.device("cuda", 0)
    round_elems = 8192 * 24
    n = round_elems * (3 * world + 1) + 8192 * 5 + 4  # ragged global tail
    full = ops.fill_synthetic("i32_full", n, seed=21)
    want = torch.cumsum(full.to(torch.int64), 0).to(torch.int32)
    boxes = p2p.Mailboxes.local(world, dev, cap=256)
    pcs = [p2p.PeerCollectives(boxes[r], r, world, 256, dev) for r in range(world)]
    layout = [wd.cyclic_rounds(n, r, world, round_elems) for r in range(world)]
    rounds = layout[0][0]
    xs, wants = [], []
    for r in range(world):
        parts = layout[r][1]
        xs.append(torch.cat([full[s:s + m] for s, m in parts]))
        wants.append(torch.cat([want[s:s + m] for s, m in parts]))
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    cap = 148 // world
    torch.cuda.synchronize()
    try:
        for call in range(3):
            outs = [torch.full_like(x, -1) for x in xs]
            for r in (range(world) if call % 2 == 0 else reversed(range(world))):
                with torch.cuda.stream(streams[r]):
                    pcs[r].scan_inclusive_i32_cyclic(xs[r], outs[r], round_elems, rounds,
                                                     max_grid=cap, stream=streams[r],
                                                     input_stable=call == 2)
            torch.cuda.synchronize()
            for r in range(world):
                assert torch.equal(outs[r], wants[r]), (call, r)
        assert not any(pc.failed() for pc in pcs)
    finally:
        torch.cuda.synchronize()
        boxes[0].close()


def test_cyclic_scan_missing_peer_fails_loudly(mods):
    """A rank whose peer never launches its half of the cyclic scan: the
    sweeper's polls time out ONCE (not once per round), the kernel completes,
    the rank's error word is set, and the device stays usable."""
    import time
    ops, p2p, wd = mods
    dev = torch.device("cuda", 0)
    round_elems = 8192 * 4
    n = round_elems * 2 * 6
    full = ops.fill_synthetic("i32_full", n, seed=5)
    boxes = p2p.Mailboxes.local(2, dev, cap=64)
    pcs = [p2p.PeerCollectives(boxes[r], r, 2, 64, dev) for r in range(2)]
    rounds, parts = wd.cyclic_rounds(n, 1, 2, round_elems)
    x = torch.cat([full[s:s + m] for s, m in parts])
    torch.cuda.synchronize()
    try:
        t0 = time.perf_counter()
        pcs[1].scan_inclusive_i32_cyclic(x, round_elems=round_elems, rounds=rounds)
        torch.cuda.synchronize()
        elapsed = time.perf_counter() - t0
        assert pcs[1].failed()
        assert elapsed < 30.0, elapsed  # one ~4 s timeout, not one per round
        # the GPU is still fine
        y = ops.scan_inclusive_i32(x)
        assert torch.equal(y, torch.cumsum(x.to(torch.int64), 0).to(torch.int32))
    finally:
        torch.cuda.synchronize()
        boxes[0].close()


def _child_read_mailbox(handle: bytes, world: int, q) -> None:
    import ctypes as C
    import torch as T
    from paper_2112_10034_b200 import _lib
    T.cuda.set_device(0)
    lib = _lib.load()
    p = C.c_void_p()
    rc = lib.wf_ipc_open(C.create_string_buffer(handle, 64), C.byref(p))
    if rc != 0:
        q.put(("error", _lib.last_error()))
        return
    out = T.zeros(1, dtype=T.int64, device="cuda")
    rc = lib.wf_fold_u64(p, 2 * world, out.data_ptr(), None)
    T.cuda.synchronize()
    q.put(("ok", int(out.item())) if rc == 0 else ("error", _lib.last_error()))
    lib.wf_ipc_close(p)


def test_mailbox_ipc_mapping_across_processes(mods):
    """The parent writes a pattern into its mailbox; a spawned process maps
    it with wf_ipc_open (the multi-process path of Mailboxes) and reads it
    back with a kernel."""
    import ctypes as C
    from paper_2112_10034_b200 import _lib
    lib = _lib.load()
    world = 4
    box = C.c_void_p()
    assert lib.wf_mailbox_alloc(world, C.byref(box)) == 0
    try:
        vals = torch.arange(1, 2 * world + 1, dtype=torch.int64, device="cuda") * 1000003
        for i in range(2 * world):  # one-element folds = device copies into the slots
            assert lib.wf_fold_u64(C.c_void_p(vals.data_ptr() + 8 * i), 1,
                                   C.c_void_p(box.value + 8 * i), None) == 0
        torch.cuda.synchronize()
        handle = (C.c_char * 64)()
        assert lib.wf_ipc_handle(box, handle) == 0, _lib.last_error()
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        proc = ctx.Process(target=_child_read_mailbox, args=(bytes(handle), world, q))
        proc.start()
        status, value = q.get(timeout=180)
        proc.join(timeout=60)
        assert status == "ok", value
        assert value == int(vals.sum().item())
    finally:
        lib.wf_mailbox_free(box)


def _rank_main(rank: int, world: int, port: int, n: int, q) -> None:
    import os
    import torch as T
    import torch.distributed as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    T.cuda.set_device(0)
    D.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2112_10034_b200 import distributed as wd, ops, p2p
        dev = T.device("cuda", 0)
        shards = [wd.shard_range(n, r, world) for r in range(world)]
        xs = [ops.fill_synthetic("f32_unit", hi - lo, seed=11, base=lo, device=dev)
              for lo, hi in shards]
        want = ops.fold(T.cat([ops.reduce_sum_f32(x) for x in xs]))  # NCCL-path combine, locally
        pr = p2p.PeerReducer.for_process_group(dev)
        got = [pr.reduce_sum_f32(xs[rank]).clone() for _ in range(3)]
        pc = p2p.PeerCollectives.for_process_group(dev, cap=256)
        xi = ops.fill_synthetic("i32_full", 5000 + rank, seed=rank, device=dev)
        carry = pc.exscan_u32(ops.reduce_sum_i32(xi))
        xu = ops.fill_synthetic("u8_uniform", 777, seed=rank, device=dev)
        bins = pc.allreduce_u64(ops.histogram256_u8(xu))
        carry_fused = pc.reduce_exscan_i32(xi)     # K1 + exchange in one kernel
        bins_fused = pc.histogram256_u8(xu)        # K5 + all-reduce in one kernel
        _, c3 = pc.compact_gt0_i32(xi)             # K4 + offsets in one kernel
        T.cuda.synchronize()
        res = [bool(T.equal(g.view(T.int32), want.view(T.int32))) for g in got]
        res.append(not pc.failed())
        res.append(int(bins.sum().item()) == 777 * world)
        totals = [int(ops.reduce_sum_i32(ops.fill_synthetic("i32_full", 5000 + r, seed=r,
                                                              device=dev)).item()) & 0xFFFFFFFF
                  for r in range(world)]
        res.append((int(carry[0].item()) & 0xFFFFFFFF) == (sum(totals[:rank]) & 0xFFFFFFFF))
        res.append(bool(T.equal(carry_fused, carry)) and bool(T.equal(bins_fused, bins))
                   and not pc.failed())
        cnts = [int((ops.fill_synthetic("i32_full", 5000 + r, seed=r, device=dev) > 0).sum())
                for r in range(world)]
        res.append(c3.tolist() == [cnts[rank], sum(cnts[:rank]), sum(cnts)])
        q.put((rank, res))
        D.barrier()
        pr.close()
        pc.close()
    except Exception as e:  # reported to the parent
        q.put((rank, f"{type(e).__name__}: {e}"))
    finally:
        D.destroy_process_group()


def test_peer_reducer_two_processes_one_gpu(mods):
    """The real multi-process path (mailbox export, IPC open, consensus,
    fused kernel) with two ranks sharing one GPU: their kernels time-slice
    rather than run concurrently, so each waits for the other's context —
    slow, but the protocol and the result are the multi-GPU ones."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, (1 << 20) + 33, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == [True] * 8 and res[1] == [True] * 8, res


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_peer_collectives_in_process(mods, world):
    """wf_peer_exchange with `world` ranks as concurrent single-block kernels
    on one GPU: scan carries (u32, wrapping), compaction offsets (u64) and the
    bin all-reduce, over several epochs (both mailbox banks), results
    identical on every rank and equal to the host-side combine."""
    ops, p2p, wd = mods
    dev = torch.device("cuda", 0)
    cap = 256
    boxes = p2p.Mailboxes.local(world, dev, cap=cap)
    pcs = [p2p.PeerCollectives(boxes[r], r, world, cap, dev) for r in range(world)]
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    rng = np.random.default_rng(world)
    try:
        for step in range(4):
            u32 = rng.integers(-2**31, 2**31, size=world, dtype=np.int64).astype(np.int32)
            u64 = rng.integers(0, 2**40, size=world, dtype=np.int64)
            vec = rng.integers(0, 2**33, size=(world, cap), dtype=np.int64)
            ins = [(torch.tensor(u32[r:r + 1], device=dev), torch.tensor(u64[r:r + 1], device=dev),
                    torch.tensor(vec[r], device=dev)) for r in range(world)]
            torch.cuda.synchronize()
            outs = [None] * world
            order = range(world) if step % 2 == 0 else reversed(range(world))
            for r in order:
                with torch.cuda.stream(streams[r]):
                    a, b, c = ins[r]
                    outs[r] = (pcs[r].exscan_u32(a, stream=streams[r]),
                               pcs[r].exscan_u64(b, stream=streams[r]),
                               pcs[r].allreduce_u64(c, stream=streams[r]))
            torch.cuda.synchronize()
            w32 = u32.astype(np.uint32).astype(np.uint64)
            for r in range(world):
                assert not pcs[r].failed()
                e32, e64, red = (t.cpu().numpy() for t in outs[r])
                assert e32.view(np.uint32).tolist() == [int(w32[:r].sum()) & 0xFFFFFFFF,
                                                        int(w32.sum()) & 0xFFFFFFFF]
                assert e64.tolist() == [int(u64[:r].sum()), int(u64.sum())]
                assert np.array_equal(red, vec.sum(0))
    finally:
        torch.cuda.synchronize()
        boxes[0].close()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_fused_peer_kernels_in_process(mods, world):
    """K1 + scan-carry exchange, K4 + offset exchange and K5 + bin all-reduce
    fused into one kernel per rank (wf_reduce_sum_i32_exscan_mg,
    wf_compact_gt0_i32_mg, wf_histogram256_u8_mg): `world`
    concurrent ranks on one GPU, several epochs interleaved with the
    stand-alone exchange on the same mailbox, results identical on every rank
    and equal to the per-rank kernels combined on the host."""
    ops, p2p, wd = mods
    dev = torch.device("cuda", 0)
    cap = 256
    boxes = p2p.Mailboxes.local(world, dev, cap=cap)
    pcs = [p2p.PeerCollectives(boxes[r], r, world, cap, dev) for r in range(world)]
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    n_i, n_u = (1 << 22) * world + 977, (1 << 24) * world + 33
    si = [wd.shard_range(n_i, r, world) for r in range(world)]
    su = [wd.shard_range(n_u, r, world) for r in range(world)]
    xs = [ops.fill_synthetic("i32_full", hi - lo, seed=5, base=lo) for lo, hi in si]
    us = [ops.fill_synthetic("u8_uniform", hi - lo, seed=6, base=lo) for lo, hi in su]
    totals = [int(ops.reduce_sum_i32(x).item()) & 0xFFFFFFFF for x in xs]
    want_bins = sum(ops.histogram256_u8(u) for u in us)
    want_sel = [x[x > 0] for x in xs]
    counts = [int(w.numel()) for w in want_sel]
    # created up front: a pageable H2D copy inside the loop would block the
    # host behind this rank's spinning kernel before the next rank launches
    offs_in = [torch.tensor([r + 1], device=dev) for r in range(world)]
    torch.cuda.synchronize()
    try:
        for step in range(4):
            outs = [None] * world
            order = range(world) if step % 2 == 0 else reversed(range(world))
            for r in order:
                with torch.cuda.stream(streams[r]):
                    c = pcs[r].reduce_exscan_i32(xs[r], stream=streams[r])
                    off = pcs[r].exscan_u64(offs_in[r], stream=streams[r])
                    b = pcs[r].histogram256_u8(us[r], stream=streams[r])
                    co, c3 = pcs[r].compact_gt0_i32(xs[r], stream=streams[r])
                    outs[r] = (c, off, b, co, c3)
            torch.cuda.synchronize()
            for r in range(world):
                c, off, b, co, c3 = outs[r]
                assert not pcs[r].failed(), (step, r)
                assert (int(c[0]) & 0xFFFFFFFF, int(c[1]) & 0xFFFFFFFF) == (
                    sum(totals[:r]) & 0xFFFFFFFF, sum(totals) & 0xFFFFFFFF), (step, r)
                assert off.tolist() == [r * (r + 1) // 2, world * (world + 1) // 2]
                assert torch.equal(b, want_bins), (step, r)
                assert c3.tolist() == [counts[r], sum(counts[:r]), sum(counts)], (step, r)
                assert torch.equal(co[:counts[r]], want_sel[r]), (step, r)
    finally:
        torch.cuda.synchronize()
        boxes[0].close()
