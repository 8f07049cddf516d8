#!/usr/bin/env python
"""Benchmark of the B200 warp-primitive path (BASELINE.json metric:
"Gelem/s + HBM GB/s (% of peak) per warp kernel at 1/2/4/8 B200 vs CPU ref").

Headline workload (one JSON line, `value`): BASELINE config 2 — fp32
warp-shuffle reduction over 2^30 elements, sharded across the N ranks
(strong scaling), per-GPU partials combined by an NCCL all-gather and a
fixed-order fold.  A step = one pass of the hot path over the whole 2^30
input.  `per_kernel` adds the other BASELINE configs measured in the same run
(C1 on rank 0 only; C3-C5 sharded like C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N>1) every rank drives one GPU; times are CUDA-event times
on each rank's stream, max over ranks.  `--impl reference` times the CPU
restatement of the reference's collapsed loop nests (oracle/collapse_ref.c,
the reference itself is pure Python and is not installed on the GPU box) on
the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Gelem/s + HBM GB/s (% of peak) per warp kernel at 1/2/4/8 B200 vs CPU ref"
N_C1 = 1 << 20
N_C2 = 1 << 30
N_C3 = 1 << 28
N_C4 = 1 << 28
N_C5 = 1 << 32
# C2 does not pin a block size (C1 does: 256).  Back-to-back steps at 2^30:
# 256-thread CTAs 615 us, 512 598 us from the first steps on, 1024 587 us but
# only after ~25 launches (606-612 before; tools/bench_loop_probe2.py,
# profiles/r01_reduce_experiments.md) — 512 is the robust choice.
BLOCK_C2 = int(os.environ.get("WF_BENCH_BLOCK_C2", "256"))
# timed steps (headline and C3-C5) as programmatic dependent launches
# (WF_FLAG_INPUT_STABLE: consecutive steps read one input that nothing
# between them writes); WF_BENCH_PDL=0 measures plain stream-ordered launches
PDL_STEPS = os.environ.get("WF_BENCH_PDL", "1") != "0"
# C3 at N > 1: super-tile (round) size of the block-cyclic layout — 512 tiles,
# a third of one GPU's on-chip pipeline (1776 tiles), so a rank keeps reading
# while the lower ranks' round totals arrive
C3_ROUND = 1 << 22
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
NOMINAL_HBM_GBS = 8000.0   # north_star / BASELINE.md §4: % of peak also vs 8.0 TB/s


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        v = float(json.loads(p.read_text())["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs, torch copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(name: str):
    """dram bytes per launch of `name` from the committed ncu --set full
    summary (profiles/ncu_traffic.json), or None."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        return d.get(name)
    except Exception:
        return None


# ---- clocks sampling (B200_PROFILING.md "clocks DURING the timed region") --
class ClockSampler:
    """Polls NVML (SM clock + clock-event reasons) every ~2 ms in a thread for
    the duration of the timed region; falls back to `nvidia-smi -lms 100`."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.max_mhz = None
        self._stop = None
        self._thread = None
        self._nvml = None

    def _handle(self, nv):
        import torch
        try:  # map the CUDA device to its NVML handle through the PCI address
            pr = torch.cuda.get_device_properties(self.dev)
            bus_id = f"{int(pr.pci_domain_id):08x}:{int(pr.pci_bus_id):02x}:{int(pr.pci_device_id):02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus_id.encode())
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.dev)

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = self._handle(nv)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._nvml = nv
            self._stop = threading.Event()

            def poll():
                while not self._stop.is_set():
                    try:
                        mhz = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(mhz), int(rs)))
                    except Exception:
                        pass
                    self._stop.wait(0.002)
            self._thread = threading.Thread(target=poll, daemon=True)
            self._thread.start()
            time.sleep(0.01)
        except Exception:
            self._nvml = None
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0}
        reasons = sorted({name for _, rs in self.samples for bit, name in self.REASONS.items()
                          if rs & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "source": "NVML, ~2 ms polling during the timed loop"}


# ---- distributed plumbing --------------------------------------------------
def init_dist(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only: every rank on GPU 0 over gloo, to run the N>1 code path
    # (IPC mailboxes, fused exchanges) as real processes on a 1-GPU box
    same_gpu = os.environ.get("WF_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    if args.impl == "ours" and local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local}, but only "
                         f"{torch.cuda.device_count()} visible")
    if world > 1:
        torch.cuda.set_device(local) if args.impl == "ours" else None
        backend = "nccl" if args.impl == "ours" and not same_gpu else "gloo"
        backend = os.environ.get("WF_BENCH_BACKEND", backend)
        dist.init_process_group(backend=backend,
                                device_id=torch.device("cuda", local) if backend == "nccl" else None)
    elif args.impl == "ours":
        torch.cuda.set_device(0)
    return rank, world, local


def barrier_sync(world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_sum(t, world: int):
    """Sum of a small device tensor over ranks (identity at N=1)."""
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def all_gather_small(t, world: int):
    """[world, *t.shape] of a small per-rank device tensor."""
    from paper_2112_10034_b200 import distributed as wd
    return wd.exchange(t) if world > 1 else t.reshape(1, *t.shape)


# ---- result checks (after each timed region; not timed) --------------------
# Every number this file prints comes from a run whose result is checked
# against an independent torch computation on the same device data.
def _wrap32(v: int) -> int:
    return ((int(v) + (1 << 31)) % (1 << 32)) - (1 << 31)


def check_c2(got, x, world: int, n_total: int) -> bool:
    """fp32 sum within the SURVEY §8c bound 2*ceil(log2 n)*2^-24*sum|x| of
    the fp64 sum, and identical on every rank."""
    import math
    import torch
    ex = torch.stack([torch.sum(x, dtype=torch.float64), torch.sum(x.abs(), dtype=torch.float64)])
    ex = all_sum(ex, world)
    exact, absx = float(ex[0]), float(ex[1])
    tol = 2 * math.ceil(math.log2(n_total)) * 2.0 ** -24 * absx
    same = bool((all_gather_small(got.view(torch.int32), world) == got.view(torch.int32)).all())
    return abs(float(got.item()) - exact) <= tol and same


def check_c1(got, x) -> bool:
    import torch
    return int(got.item()) == _wrap32(int(torch.sum(x.to(torch.int64))))


def check_c3(y, x, world: int, rank: int) -> bool:
    """Inclusive scan of the shard with the global carry: first element,
    every first difference (mod 2^32) and the last element."""
    import torch
    tot = torch.sum(x.to(torch.int64)).reshape(1)
    totals = all_gather_small(tot, world).reshape(-1).tolist()
    carry = _wrap32(sum(totals[:rank]))
    ok = int(y[0]) == _wrap32(carry + int(x[0]))
    ok &= int(y[-1]) == _wrap32(carry + totals[rank])
    step = 1 << 26
    for lo in range(1, x.numel(), step):
        hi = min(x.numel(), lo + step)
        d = (y[lo:hi].to(torch.int64) - y[lo - 1:hi - 1].to(torch.int64)
             - x[lo:hi].to(torch.int64)) % (1 << 32)
        ok &= int(d.count_nonzero()) == 0
    return bool(all_sum(torch.tensor([0 if ok else 1], device=x.device), world).item() == 0)


def check_c3_cyclic(y, parts, world: int) -> bool:
    """Block-cyclic scan: this rank's output == the global inclusive scan
    (the whole synthetic array regenerated here, int64 cumsum wrapped to
    int32) at its super-tiles' positions."""
    import torch
    from paper_2112_10034_b200 import ops
    full = ops.fill_synthetic("i32_full", N_C3, seed=0, device=y.device)
    want = torch.cumsum(full.to(torch.int64), 0).to(torch.int32)
    del full
    ok, off = True, 0
    for start, m in parts:
        ok &= torch.equal(y[off:off + m], want[start:start + m])
        off += m
    del want
    return bool(all_sum(torch.tensor([0 if ok else 1], device=y.device), world).item() == 0)


def check_c4(res, x, world: int, rank: int) -> bool:
    """Ordered compaction == masked_select of the shard; offset / total ==
    exclusive / full sums of the per-rank counts."""
    import torch
    out, count = res[0], res[1]
    m = int(count.item())
    want = torch.masked_select(x, x > 0)
    ok = m == want.numel() and torch.equal(out[:m], want)
    counts = all_gather_small(torch.tensor([want.numel()], dtype=torch.int64, device=x.device),
                              world).reshape(-1).tolist()
    if world > 1:
        ok &= int(res[2].item()) == sum(counts[:rank]) and int(res[3].item()) == sum(counts)
    return bool(all_sum(torch.tensor([0 if ok else 1], device=x.device), world).item() == 0)


def check_c5(bins, u, world: int) -> bool:
    """All-reduced bins == all-reduced torch.bincount of the shard (16 slices)."""
    import torch
    want = torch.zeros(256, dtype=torch.int64, device=u.device)
    step = (u.numel() + 15) // 16
    for lo in range(0, u.numel(), step):
        want += torch.bincount(u[lo:lo + step].to(torch.int32), minlength=256)
    want = all_sum(want, world)
    ok = torch.equal(bins.view(torch.int64), want)
    return bool(all_sum(torch.tensor([0 if ok else 1], device=u.device), world).item() == 0)


# ---- CPU baselines (oracle port of the collapsed loop nests) ---------------
CPU_POOL_LOG2 = 27    # 512 MiB fp32 pool: DRAM-resident like the real 4 GiB input
CPU_SLICE_LOG2 = 24   # one bounded sample = one 2^24-element slice of the pool


def _cpu_c2_pool():
    """The C2 workload's first 2^27 synthetic fp32 elements.  Samples rotate
    through 2^24-element slices of it so every sample streams from DRAM (a
    single cache-resident slice overstated the CPU rate ~2x: 5.85 vs 2.76
    Gelem/s on the B200 box's host)."""
    from oracle import synthetic
    return synthetic.generate("f32_unit", 1 << CPU_POOL_LOG2, seed=1)


def _cpu_c2_run(pool, i: int, workers: int) -> int:
    from oracle import cref
    k = 1 << CPU_SLICE_LOG2
    s = (i % (len(pool) // k)) * k
    cref.reduce_f32(pool[s:s + k], 64 * workers, 256, workers)
    return k


def cpu_baseline_c2(budget_s: float = 10.0) -> dict:
    """The reference's per-warp-partials f32 reduction, collapsed into
    block/warp/lane loop nests (oracle/collapse_ref.c), on all host threads;
    repeated over rotating DRAM-resident slices until ~budget_s."""
    from oracle import cref
    cref.build()
    workers = cref.workers_default()
    pool = _cpu_c2_pool()
    _cpu_c2_run(pool, 0, workers)  # warm
    reps, elems, t0 = 0, 0, time.perf_counter()
    while True:
        elems += _cpu_c2_run(pool, reps + 1, workers)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or reps >= 100000:
            break
    return {"value": round(elems / el / 1e9, 6), "unit": "Gelem/s", "cores": workers,
            "kind": "port",
            "sample": f"{reps} x 2^{CPU_SLICE_LOG2} fp32 slices rotating through a "
                      f"2^{CPU_POOL_LOG2}-element DRAM-resident pool (collapse_ref.c "
                      f"per-warp-partials shfl_down reduction, grid {64 * workers} x block 256, "
                      f"{workers} threads, {el:.1f} s)"}


_CPU_POOLS: dict = {}


def _cpu_pool(gen: str):
    """2^27-element DRAM-resident pools (generated once per run); samples
    rotate through their 2^24-element slices, like the C2 baseline."""
    if gen not in _CPU_POOLS:
        from oracle import synthetic
        _CPU_POOLS[gen] = synthetic.generate(gen, 1 << CPU_POOL_LOG2, seed=0)
    return _CPU_POOLS[gen]


def cpu_baseline_kernel(kind: str, budget_s: float) -> dict:
    from oracle import cref, synthetic
    workers = cref.workers_default()
    k = 1 << CPU_SLICE_LOG2
    if kind == "c1":  # the whole C1 input is 4 MiB: it is cache-resident on the CPU too
        x = synthetic.generate("i32_full", N_C1, seed=0)
        fn, n, note = (lambda i: cref.reduce_i32(x, 8 * workers, 256, workers)), N_C1, ""
    else:
        pool = _cpu_pool("u8_uniform" if kind == "c5" else "i32_full")
        slices = len(pool) // k
        run = {"c3": lambda v: cref.scan_i32(v, 256, workers),
               "c4": lambda v: cref.compact_gt0_i32(v, 256, workers),
               "c5": lambda v: cref.hist256_u8(v, 64 * workers, 256, workers)}[kind]
        fn = lambda i: run(pool[(i % slices) * k:(i % slices + 1) * k])  # noqa: E731
        n = k
        note = f" (slices rotating through a 2^{CPU_POOL_LOG2}-element DRAM-resident pool)"
    fn(0)
    reps, t0 = 0, time.perf_counter()
    while True:
        fn(reps + 1)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or reps >= 100000:
            break
    ref_path = {
        "c1": "the reference runs this kernel (SURVEY 8c per-warp-partials text); this is "
              "its collapsed loop nest in C",
        "c3": "the reference expresses only the in-warp prefix (lane-reversed shfl_down); "
              "block/grid carries are this C restatement's",
        "c4": "none: not expressible in the reference DSL (no ballot/atomics, "
              "dsl/lexer.py:18-25); a C restatement of the CUDA semantics",
        "c5": "none: not expressible in the reference DSL (no u8/atomics, "
              "dsl/parser.py:83-88); a C restatement of the CUDA semantics"}[kind]
    return {"value": round(n * reps / el / 1e9, 6), "unit": "Gelem/s", "cores": workers,
            "kind": "port", "reference_path": ref_path,
            "sample": f"{reps} x {n} elements{note}, {el:.1f} s"}


# ---- GPU timing helpers -----------------------------------------------------
def time_launches(fn, steps: int, warmup: int, flush=None, clocks: dict | None = None,
                  world: int = 1):
    """Per-launch times (ms) on the current stream.  Without a flush the
    `steps` launches run back to back between two events (the steady state of
    a stream of calls; inputs larger than L2 need no flush) and the average
    is returned for each; with a flush (C1) every launch is bracketed by its
    own events right after the L2 flush.  `clocks`: filled with the SM clock
    summary sampled during the back-to-back loop (K5 on random bytes can hit
    the board's power cap).  `world` > 1 (a sharded leg every rank runs): a
    barrier before the warm-up and before the timed loop, so no rank's fused
    exchange waits inside the kernel for a rank still busy elsewhere (e.g.
    the rank-0-only C1 leg) and the timed loops start together."""
    import torch
    barrier_sync(world)  # whatever wrote the inputs has finished (WF_FLAG_INPUT_STABLE)
    for _ in range(warmup):
        if flush is not None:
            flush()
        fn()
    barrier_sync(world)
    if flush is None:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(torch.cuda.current_device()) as clk:
            s.record()
            for _ in range(steps):
                fn()
            e.record()
            torch.cuda.synchronize()
        if clocks is not None:
            clocks.update(clk.summary())
        return [s.elapsed_time(e) / steps] * steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for s, e in evs:
        flush()
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in evs]


def run_ours(args, rank, world, local) -> dict | None:
    import torch
    from paper_2112_10034_b200 import distributed as wd, ops

    peak, peak_src = measured_peak()
    dev = torch.device("cuda", local)
    lo, hi = wd.shard_range(N_C2, rank, world)
    n_local = hi - lo
    x = ops.fill_synthetic("f32_unit", n_local, seed=1, base=lo, device=dev)
    torch.cuda.synchronize()

    # ---- N>1: fuse the partials' exchange into K2 over peer memory --------
    peer, exchange = None, "none (1 GPU)"
    if world > 1:
        from paper_2112_10034_b200 import p2p
        lo_p, hi_p = wd.shard_range(1 << 20, rank, world)
        probe = ops.fill_synthetic("f32_unit", hi_p - lo_p, seed=7, base=lo_p, device=dev)
        peer, why = p2p.try_peer_reducer(dev, probe)
        exchange = ("peer memory, fused into K2 (CUDA IPC mailboxes over NVLink)" if peer
                    else f"NCCL all-gather + fold kernel (peer path unavailable: {why})")
        log(f"rank {rank}: partial exchange = {exchange}")

    # ---- headline: K2 step over the 2^30 job, device-resident inputs ------
    # The timed region is K back-to-back steps bracketed by two events (no
    # per-step events: they would serialise kernel boundaries that a real
    # stream of steps overlaps).  When a step is one kernel (1 GPU, or the
    # fused peer-memory exchange) the kernel's average duration IS the step
    # time; with the NCCL fallback the kernel alone is timed in a second loop.
    launches = 0

    def step():
        nonlocal launches
        # consecutive steps read the same input and nothing between them
        # writes it: each step is a programmatic dependent launch that streams
        # while the previous step drains (WF_FLAG_INPUT_STABLE; same bits)
        if peer is not None:  # one kernel: local reduce + exchange + fold
            part = peer.reduce_sum_f32(x, block=BLOCK_C2, input_stable=PDL_STEPS)
        else:
            part = ops.reduce_sum_f32(x, block=BLOCK_C2, input_stable=PDL_STEPS)
        launches += 1
        if world > 1 and peer is None:
            ops.fold(wd.exchange(part).reshape(-1))
            launches += 1
        return part

    for _ in range(args.warmup):
        step()
    launches = 0
    barrier_sync(world)
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            step()
        t1.record()
        barrier_sync(world)
    step_ms = t0.elapsed_time(t1) / args.steps
    gpu_launches = launches  # our kernels inside the timed region
    checks = {"c2_reduce_f32": check_c2(step(), x, world, N_C2)}
    if peer is not None:  # the timed exchange must still agree with the NCCL path, bit for bit
        got = peer.reduce_sum_f32(x, block=BLOCK_C2)
        want = ops.fold(wd.exchange(ops.reduce_sum_f32(x, block=BLOCK_C2)).reshape(-1))
        if not torch.equal(got.view(torch.int32), want.view(torch.int32)):
            log(f"rank {rank}: fused K2 exchange disagrees with NCCL after timing: "
                f"{float(got.item())} vs {float(want.item())}")
            exchange += " — FAILED post-timing check"
            checks["c2_reduce_f32"] = False
    if world == 1 or peer is not None:
        kern_ms, kern_timing = step_ms, "timed region / steps (one kernel per step)"
    else:
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(args.steps):
            ops.reduce_sum_f32(x, block=BLOCK_C2)
        s1.record()
        torch.cuda.synchronize()
        kern_ms, kern_timing = s0.elapsed_time(s1) / args.steps, "separate back-to-back K2 loop"
    step_ms_max = max_over_ranks(step_ms, world)
    value = N_C2 / (step_ms_max * 1e-3) / 1e9
    achieved = 4.0 * n_local / (kern_ms * 1e-3) / 1e9

    log(f"rank {rank}: headline done ({step_ms:.3f} ms/step)")
    # ---- e2e through the C-ABI host entry point ---------------------------
    host = torch.empty(n_local, dtype=torch.float32, pin_memory=True)
    host.copy_(x)
    e2e_steps = args.steps
    ops.reduce_sum_f32_host(host, device=dev)  # warm (staging + streams)
    barrier_sync(world)
    t = time.perf_counter()
    for _ in range(e2e_steps):
        v = ops.reduce_sum_f32_host(host, device=dev)
        total = torch.tensor([v], dtype=torch.float32, device=dev)
        if world > 1:  # combine the per-rank partials: all-gather + fixed-order fold
            total = ops.fold(wd.exchange(total).reshape(-1))
            float(total.item())
    e2e_ms = (time.perf_counter() - t) * 1e3 / e2e_steps
    checks["e2e"] = check_c2(total, x, world, N_C2)
    e2e_ms_max = max_over_ranks(e2e_ms, world)
    # the link's own ceiling on this box: plain pinned H2D copy of the same bytes
    dst = torch.empty_like(x)
    dst.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    dst.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    h2d_gbs = 4.0 * n_local / (time.perf_counter() - t) / 1e9
    del host, dst

    log(f"rank {rank}: e2e done")
    # ---- per-kernel lines for the other BASELINE configs -------------------
    per = {}
    if not args.headline_only:
        per = per_kernel(args, rank, world, local, dev, peak, checks)
    per["c2_reduce_f32"] = {"gelem_s": round(value, 3), "gbs": round(achieved, 1),
                            "frac_of_peak": round(achieved / peak, 4),
                            "frac_of_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
                            "kernel_us": round(kern_ms * 1e3, 2), "n": N_C2,
                            "bytes_per_elem": 4}
    del x
    torch.cuda.empty_cache()

    if rank != 0:
        return None
    predicted = None
    if world == 1 and not args.headline_only and not args.no_shards:
        log("rank 0: per-rank steps at the 1/2/4/8-GPU shard sizes (one-GPU scaling prediction)")
        from paper_2112_10034_b200 import benchmarks as bm
        rows = bm.bench_shards(iters=10, repeats=3)
        predicted = {"how": "per-rank step of each sharded config at the 1/2/4/8-GPU shard "
                            "sizes, measured on this one GPU with the fused per-rank kernels "
                            "(world-1 mailbox: the exchange protocol runs, the NVLink round "
                            "trip does not) as dependent launches; speedup = t(1) / t(N).  "
                            "A prediction: the driver's multi-GPU run measures the real curve",
                     "configs": {}}
        names = {"reduce_sum_f32": "C2", "scan_inclusive_i32": "C3", "compact_gt0_i32": "C4",
                 "histogram256_u8": "C5"}
        for r in rows:
            predicted["configs"].setdefault(names[r["op"]], {})[f"N{r['n_gpus']}"] = {
                "per_rank_us": round(r["per_rank_us"], 1),
                "speedup": round(r["predicted_speedup"], 3),
                "efficiency": round(r["predicted_efficiency"], 3)}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_c2(args.cpu_budget)
        for k, key in (("c1", "c1_reduce_i32"), ("c3", "c3_scan_i32"), ("c4", "c4_compact_i32"),
                       ("c5", "c5_hist_u8")):
            if key in per:
                per[key]["cpu_baseline"] = cpu_baseline_kernel(k, args.cpu_budget / 3)
    traffic = ncu_traffic("reduce_sum_f32")
    return {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "Gelem/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms_max, 5),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (splitmix64 index hash, generated in HBM)",
        "config": {
            "workload": "C2: fp32 warp-shuffle reduction over 2^30 elements sharded across "
                        f"{world} B200",
            "exchange": exchange,
            "n": N_C2, "block": BLOCK_C2, "parallelism": f"shard{world}",
            "launch": ("programmatic dependent launches: each timed step (headline and "
                       "per_kernel C3-C5) starts streaming its input while the previous "
                       "step drains (WF_FLAG_INPUT_STABLE); every step still reads all of "
                       "its input" if PDL_STEPS else "stream-ordered launches"),
            "l2": "inputs larger than L2 (4 GiB vs 126 MB), no flush needed",
        },
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "frac_of_nominal_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
                     "kernel": "reduce_sum_f32 (K2)", "peak_source": peak_src,
                     "kernel_timing": kern_timing,
                     "algorithmic_bytes_per_launch": 4 * n_local},
        "cpu_baseline": cpu,
        "e2e": {"value": round(N_C2 / (e2e_ms_max * 1e-3) / 1e9, 4), "unit": "Gelem/s",
                "h2d_bytes_per_step": 4 * n_local, "d2h_bytes_per_step": 4,
                "path": "wf_reduce_sum_f32_host (pinned host -> chunked H2D overlapped with K2 "
                        "-> D2H of the result)", "steps": e2e_steps,
                "association": "per-chunk K2 partials (block 512) + fixed-order fold: a "
                               "different fp32 order than the one-launch headline; both "
                               "checked against the fp64 sum within the SURVEY 8c bound",
                "pcie_h2d_gbs": round(h2d_gbs, 2),
                "frac_of_h2d_copy": round(4.0 * n_local / (e2e_ms * 1e-3) / 1e9 / h2d_gbs, 4)},
        "gpu_launches": gpu_launches,
        "verified": checks,
        "clocks": clk.summary(),
        "per_kernel": per,
        "predicted_scaling": predicted,
    }


E2E_STEPS = 5  # per-kernel e2e legs: median of 5 synchronous calls, link ceiling likewise


def e2e_host_leg(kind: str, x, checks: dict) -> dict:
    """One per-kernel e2e leg: the op through its C-ABI host entry point
    (``wf_*_host``: pinned host input -> chunked H2D overlapped with the
    kernel -> D2H into a pinned host output), timed by the host clock around
    the synchronous call, checked against the device-resident result.  The
    link ceiling is the same bytes copied by plain concurrent pinned
    H2D + D2H (two streams), so ``frac_of_link`` = that time / e2e time."""
    import torch
    from paper_2112_10034_b200 import ops
    n = x.numel()
    host = torch.empty(n, dtype=x.dtype, pin_memory=True)
    host.copy_(x)
    if kind == "scan":
        want = ops.scan_inclusive_i32(x).cpu()
        hout = torch.empty(n, dtype=torch.int32, pin_memory=True)
        call = lambda: ops.scan_inclusive_i32_host(host, hout, device=x.device)  # noqa: E731
        d2h_bytes = 4 * n
        ok = lambda r: torch.equal(hout, want)  # noqa: E731
        path = "wf_scan_inclusive_i32_host"
    elif kind == "compact":
        wo, wc = ops.compact_gt0_i32(x)
        m = int(wc.item())
        want = wo[:m].cpu()
        hout = torch.empty(n, dtype=torch.int32, pin_memory=True)
        call = lambda: ops.compact_gt0_i32_host(host, hout, device=x.device)  # noqa: E731
        d2h_bytes = 4 * m + 8
        ok = lambda r: r[1] == m and torch.equal(hout[:m], want)  # noqa: E731
        path = "wf_compact_gt0_i32_host"
    else:
        want = ops.histogram256_u8(x).cpu()
        hout = None
        call = lambda: ops.histogram256_u8_host(host, device=x.device)  # noqa: E731
        d2h_bytes = 256 * 8
        ok = lambda r: torch.equal(torch.from_numpy(r.view("int64")), want)  # noqa: E731
        path = "wf_histogram256_u8_host"
    h2d_bytes = n * x.element_size()
    r = call()  # warm (staging ring, copy streams)
    torch.cuda.synchronize()
    times = []
    for _ in range(E2E_STEPS):  # each call is synchronous: host clock around it
        t = time.perf_counter()
        r = call()
        times.append(time.perf_counter() - t)
    e2e_s = statistics.median(times)
    checks[f"e2e/{kind}"] = bool(ok(r))
    # link ceiling: concurrent plain pinned copies of the same byte counts
    dev_in = torch.empty_like(x)
    d2h_elems = max(1, d2h_bytes // 4)
    src = torch.empty(d2h_elems, dtype=torch.int32, device=x.device)
    dst = torch.empty(d2h_elems, dtype=torch.int32, pin_memory=True)
    s1, s2 = torch.cuda.Stream(device=x.device), torch.cuda.Stream(device=x.device)
    link = []
    for _ in range(E2E_STEPS):
        torch.cuda.synchronize()
        t = time.perf_counter()
        with torch.cuda.stream(s1):
            dev_in.copy_(host, non_blocking=True)
        with torch.cuda.stream(s2):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        link.append(time.perf_counter() - t)
    best = statistics.median(link)
    del dev_in, src, dst, host, hout
    return {"value": round(n / e2e_s / 1e9, 4), "unit": "Gelem/s", "path": path,
            "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
            "steps": E2E_STEPS, "ms_per_step": round(e2e_s * 1e3, 3),
            "link_copy_ms": round(best * 1e3, 3),
            "frac_of_link": round(best / e2e_s, 4),
            "link": "concurrent pinned H2D + D2H of the same bytes (two streams), median of 5 (same statistic as the e2e leg)"}


def reference_api_rows(dev, peak, steps: int, warm: int, checks: dict) -> dict:
    """The reference's OWN formulations of C1/C2/C3 (SURVEY §8c kernel
    texts, tests/golden/*.spk) through the drop-in
    ``launch(hybrid_transform(kernel, cfg), cfg, memory, args)`` — the call a
    reference user makes (runtime/launch.py:90).  The structural registry
    (dsl/patterns.py) routes them to native kernels (csrc/wf_patterns.cu).
    ``kernel_us``: CUDA events around back-to-back dispatches of the program
    on the stream; ``launch_us``: host clock around the full join-semantics
    ``launch`` (argument binding + kernel + synchronise)."""
    import torch
    import paper_2112_10034_b200 as wf
    from paper_2112_10034_b200.dsl import hybrid_transform, parse_module
    rows = {}
    specs = (  # key, kernel text, kind, n, grid, block, generator, bytes per element
        ("c1_wsum_i32", "C1_I32", "i32", N_C1, 4096, 256, "i32_full", 4),
        ("c2_wsum_f32", "C1_F32", "f32", N_C2, 4096, 256, "f32_unit", 4),
        ("c3_warp_prefix_i32", "C3_WARP_PREFIX", "i32", N_C3, N_C3 // 256, 256, "i32_full", 8),
    )
    for key, spk, kind, n, grid, block, gen, bpe in specs:
        kernel = parse_module((ROOT / "tests" / "golden" / f"{spk}.spk").read_text()).kernel()
        cfg = wf.LaunchConfig(grid_size=grid, block_size=block, warp_size=32)
        prog = hybrid_transform(kernel, cfg)
        mem = wf.DeviceMemory(dev)
        a = mem.alloc(4 * n)
        out_n = n if prog.native is not None and prog.native.n is None else grid * block // 32
        out = mem.alloc(4 * out_n)
        wf.ops.fill_synthetic(gen, n, seed=1, out=mem.device_view(a, kind))
        args = [a, out] if spk == "C3_WARP_PREFIX" else [a, out, n]
        bound = wf.bind_args(prog.params, mem, args)
        native = prog.native is not None and prog.native.applicable(cfg, bound)
        symbol = prog.native.symbol if prog.native is not None else None
        stream = torch.cuda.current_stream(dev)
        flush = None
        if key.startswith("c1"):  # 4 MiB: flush L2 as for the C1 headline row
            fb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
            flush = lambda: fb.fill_(1)  # noqa: E731
        t = time_launches(lambda: prog.native.run(cfg, bound, stream.cuda_stream), steps, warm,
                          flush=flush)
        kern_us = statistics.mean(t) * 1e3
        wf.launch(prog, cfg, mem, args)  # warm
        t0 = time.perf_counter()
        reps = max(3, min(steps, 20))
        for _ in range(reps):
            wf.launch(prog, cfg, mem, args)
        launch_us = (time.perf_counter() - t0) / reps * 1e6
        # check: native result == the generic compiled kernel of the same text
        got = mem.device_view(out, kind)[:out_n].clone()
        prog.native = None
        wf.launch(prog, cfg, mem, args)
        want = mem.device_view(out, kind)[:out_n]
        checks[f"reference_api/{key}"] = bool(native and torch.equal(got.view(torch.int32),
                                                                     want.view(torch.int32)))
        gbs = bpe * n / (kern_us * 1e-6) / 1e9
        rows[key] = {"kernel_text": f"tests/golden/{spk}.spk", "n": n, "grid": grid,
                     "block": block, "native_symbol": symbol,
                     "registry_hit": native,
                     "kernel_us": round(kern_us, 2), "gelem_s": round(n / kern_us / 1e3, 2),
                     "gbs": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4),
                     "launch_us": round(launch_us, 1),
                     "bytes_per_elem": bpe,
                     "l2": "flushed before every launch" if flush else "inputs larger than L2"}
        if spk != "C3_WARP_PREFIX":
            rows[key]["output"] = (f"{grid * block // 32} per-warp partials (the reference's "
                                   f"host fold of them is not timed)")
        del mem, got, want
        torch.cuda.empty_cache()
    return rows


def per_kernel(args, rank, world, local, dev, peak, checks: dict) -> dict:
    import torch
    from paper_2112_10034_b200 import distributed as wd, ops
    res = {}
    pc, exchange = None, None
    if world > 1:  # C3-C5 exchanges over peer memory when every rank can map every mailbox
        from paper_2112_10034_b200 import p2p
        pc, why = p2p.try_peer_collectives(dev)
        exchange = ("peer memory, fused into the producing kernel (C3: scan pass 1, "
                    "C4: compaction, C5: histogram)" if pc
                    else f"NCCL (peer path unavailable: {why})")
        log(f"rank {rank}: C3-C5 exchange = {exchange}")
    steps, warm = max(5, args.steps), max(3, args.warmup)

    def stats(times_ms, n_elems, bytes_per_elem, n_total, all_ranks=True):
        # all_ranks=False for legs only rank 0 runs (C1): a collective there
        # would pair with another leg's collective on the other ranks
        ms = statistics.mean(times_ms)
        ms_max = max_over_ranks(ms, world) if all_ranks else ms
        gbs = bytes_per_elem * n_elems / (ms * 1e-3) / 1e9
        return {"gelem_s": round(n_total / (ms_max * 1e-3) / 1e9, 3), "gbs": round(gbs, 1),
                "frac_of_peak": round(gbs / peak, 4),
                "frac_of_8tbs": round(gbs / NOMINAL_HBM_GBS, 4),
                "kernel_us": round(ms * 1e3, 2),
                "n": n_total, "bytes_per_elem": bytes_per_elem}

    # C1 (single GPU by definition): 2^20 int32, block 256, L2 flushed
    if rank == 0:
        x1 = ops.fill_synthetic("i32_full", N_C1, seed=0, device=dev)
        flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        t = time_launches(lambda: ops.reduce_sum_i32(x1, block=256), steps, warm,
                          flush=lambda: flush_buf.fill_(1))
        res["c1_reduce_i32"] = stats(t, N_C1, 4, N_C1, all_ranks=False)
        checks["c1_reduce_i32"] = check_c1(ops.reduce_sum_i32(x1, block=256), x1)
        res["c1_reduce_i32"]["l2"] = "flushed (256 MiB write) before every launch"
        res["c1_reduce_i32"]["bound"] = ("latency: 4 MiB is 0.6 us of HBM time; see "
                                         "latency_context_us for the launch + atomic floor")
        # latency context for this 4 MiB (0.6 us of HBM time) kernel, same
        # flushed methodology: K1 on 4 elements (launch + one atomic) and the
        # library reduction torch.sum of the same input
        tiny = x1[:4]
        t0 = time_launches(lambda: ops.reduce_sum_i32(tiny, block=256), steps, warm,
                           flush=lambda: flush_buf.fill_(1))
        tl = time_launches(lambda: torch.sum(x1), steps, warm, flush=lambda: flush_buf.fill_(1))
        res["c1_reduce_i32"]["latency_context_us"] = {
            "k1_on_4_elements": round(statistics.mean(t0) * 1e3, 2),
            "torch_sum_same_input": round(statistics.mean(tl) * 1e3, 2)}
        # end to end through the C-ABI host entry point (pinned host buffer ->
        # H2D -> K1 -> D2H of the sum), the call a reference user makes
        host1 = torch.empty(N_C1, dtype=torch.int32, pin_memory=True)
        host1.copy_(x1)
        want1 = int(ops.reduce_sum_i32(x1, block=256).item())
        got1 = ops.reduce_sum_i32_host(host1, device=dev)  # warm (staging, streams)
        e2e_t = []
        for _ in range(max(20, steps)):
            t1 = time.perf_counter()
            got1 = ops.reduce_sum_i32_host(host1, device=dev)
            e2e_t.append(time.perf_counter() - t1)
        checks["e2e/c1"] = got1 == want1
        e2e_s = statistics.median(e2e_t)
        res["c1_reduce_i32"]["e2e"] = {
            "value": round(N_C1 / e2e_s / 1e9, 4), "unit": "Gelem/s",
            "path": "wf_reduce_sum_i32_host", "h2d_bytes_per_step": 4 * N_C1,
            "d2h_bytes_per_step": 4, "ms_per_step": round(e2e_s * 1e3, 4),
            "steps": len(e2e_t), "how": "median of synchronous calls, host clock"}
        del host1
        # warm L2 (SURVEY §8d asks for cold and warm): the 4 MiB input stays
        # L2-resident and 20 launches are replayed from one CUDA graph, so
        # neither host launch cost nor HBM is in the number
        gs = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(gs):
            ops.reduce_sum_i32(x1, block=256)  # workspace for this stream
        gs.synchronize()
        graph, per_graph = torch.cuda.CUDAGraph(), 20
        with torch.cuda.graph(graph, stream=gs):
            for _ in range(per_graph):
                ops.reduce_sum_i32(x1, block=256)
        graph.replay()
        torch.cuda.synchronize()
        gt = time_launches(graph.replay, steps, warm)
        warm_us = statistics.mean(gt) * 1e3 / per_graph
        res["c1_reduce_i32"]["warm_l2"] = {
            "kernel_us": round(warm_us, 2), "gelem_s": round(N_C1 / warm_us / 1e3, 1),
            "gbs": round(4 * N_C1 / warm_us / 1e3, 1),
            "how": f"{per_graph} launches per CUDA graph replay, input L2-resident"}
        del graph
        del x1, flush_buf, tiny
    log(f"rank {rank}: C3")
    # C3 scan.  N > 1 with peer memory and a GPU per rank: block-cyclic
    # super-tiles and the single-pass cross-rank scan (8 B/elem); otherwise
    # contiguous shards and reduce-then-scan (12 B/elem at N > 1)
    lo, hi = wd.shard_range(N_C3, rank, world)
    cyclic = world > 1 and pc is not None and (
        os.environ.get("WF_BENCH_SAME_GPU") != "1" or os.environ.get("WF_BENCH_CYCLIC") == "1")
    if cyclic:
        rounds, parts = wd.cyclic_rounds(N_C3, rank, world, C3_ROUND)
        x = torch.empty(sum(m for _, m in parts), dtype=torch.int32, device=dev)
        off = 0
        for start, m in parts:  # this rank's super-tiles of the global synthetic array
            ops.fill_synthetic("i32_full", m, seed=0, base=start, out=x[off:off + m])
            off += m
        y = torch.empty_like(x)
        scan = lambda: pc.scan_inclusive_i32_cyclic(  # noqa: E731
            x, y, C3_ROUND, rounds, input_stable=PDL_STEPS)
    else:
        x = ops.fill_synthetic("i32_full", hi - lo, seed=0, base=lo, device=dev)
        y = torch.empty_like(x)
        scan = lambda: wd.scan_inclusive_i32(x, y, peer=pc, input_stable=PDL_STEPS)  # noqa: E731
    clk = {}
    t = time_launches(scan, steps, warm, clocks=clk, world=world)
    res["c3_scan_i32"] = stats(t, x.numel(), 8 if world == 1 or cyclic else 12, N_C3)
    res["c3_scan_i32"]["clocks"] = clk
    res["c3_scan_i32"]["layout"] = (
        f"block-cyclic super-tiles of {C3_ROUND} elements, single-pass scan with the round "
        f"totals all-gathered inside the kernel (8 B/elem)" if cyclic else
        "contiguous shards" + (", reduce-then-scan with a fused carry exchange (12 B/elem)"
                               if world > 1 else ""))
    if cyclic:
        checks["c3_scan_i32"] = check_c3_cyclic(scan(), parts, world)
        # C4 / C5 use contiguous shards
        x = ops.fill_synthetic("i32_full", hi - lo, seed=0, base=lo, device=dev)
    else:
        checks["c3_scan_i32"] = check_c3(scan(), x, world, rank)
    log(f"rank {rank}: C4")
    # C4 compaction
    out = torch.empty_like(x)
    compact = lambda: wd.compact_gt0_i32(x, out, peer=pc, input_stable=PDL_STEPS)  # noqa: E731
    clk = {}
    t = time_launches(compact, steps, warm, clocks=clk, world=world)
    res["c4_compact_i32"] = stats(t, hi - lo, 6, N_C4)
    res["c4_compact_i32"]["clocks"] = clk
    checks["c4_compact_i32"] = check_c4(compact(), x, world, rank)
    res["c4_compact_i32"]["bytes_per_elem_note"] = "4 B read + 4 B x selectivity (~0.5) written"
    # also 0 %, 1 % and 100 % selectivity (same n, i32_select)
    variants = {}
    for permille in (0, 10, 1000):
        ops.fill_synthetic("i32_select", hi - lo, seed=0, base=lo, param=permille, out=x)
        t = time_launches(compact, steps, warm, world=world)
        ms = statistics.mean(t)
        bpe = 4 + 4 * permille / 1000
        checks[f"c4_compact_i32/{permille / 10:g}%"] = check_c4(compact(), x, world, rank)
        variants[f"{permille / 10:g}%"] = {
            "kernel_us": round(ms * 1e3, 2),
            "gbs": round(bpe * (hi - lo) / (ms * 1e-3) / 1e9, 1),
            "gelem_s": round(N_C4 / (max_over_ranks(ms, world) * 1e-3) / 1e9, 3)}
    res["c4_compact_i32"]["selectivity_variants"] = variants
    if world == 1 and not args.headline_only:
        # end to end through the C-ABI host entry points (pinned host in and
        # out, chunked H2D / kernel / D2H ring), beside the link's own ceiling
        ops.fill_synthetic("i32_full", hi - lo, seed=0, base=lo, out=x)
        res["c3_scan_i32"]["e2e"] = e2e_host_leg("scan", x, checks)
        res["c4_compact_i32"]["e2e"] = e2e_host_leg("compact", x, checks)
    del x, y, out
    torch.cuda.empty_cache()
    log(f"rank {rank}: C5")
    # C5 histogram
    lo, hi = wd.shard_range(N_C5, rank, world)
    u = ops.fill_synthetic("u8_uniform", hi - lo, seed=0, base=lo, device=dev)
    hist = lambda: wd.histogram256_u8(u, peer=pc, input_stable=PDL_STEPS)  # noqa: E731
    clk = {}
    t = time_launches(hist, steps, warm, clocks=clk, world=world)
    res["c5_hist_u8"] = stats(t, hi - lo, 1, N_C5)
    res["c5_hist_u8"]["clocks"] = clk
    checks["c5_hist_u8"] = check_c5(hist(), u, world)
    # also all-same-value and skewed (geometric) bytes
    variants = {}
    for gen in ("u8_const", "u8_geom"):
        ops.fill_synthetic(gen, hi - lo, seed=0, base=lo, out=u)
        clk = {}
        t = time_launches(hist, steps, warm, clocks=clk, world=world)
        ms = statistics.mean(t)
        checks[f"c5_hist_u8/{gen}"] = check_c5(hist(), u, world)
        variants[gen] = {"kernel_us": round(ms * 1e3, 2),
                         "gbs": round((hi - lo) / (ms * 1e-3) / 1e9, 1),
                         "gelem_s": round(N_C5 / (max_over_ranks(ms, world) * 1e-3) / 1e9, 3),
                         "clocks": clk}
    res["c5_hist_u8"]["data_variants"] = variants
    if world == 1 and not args.headline_only:
        ops.fill_synthetic("u8_uniform", hi - lo, seed=0, base=lo, out=u)
        res["c5_hist_u8"]["e2e"] = e2e_host_leg("hist", u, checks)
    if exchange is not None:
        if pc is not None and pc.failed():  # a peer never arrived in some call: results invalid
            log(f"rank {rank}: a peer-memory exchange timed out during the C3-C5 runs")
            exchange += " — FAILED (peer timeout)"
        for k in ("c3_scan_i32", "c4_compact_i32", "c5_hist_u8"):
            res[k]["exchange"] = exchange
        if cyclic:
            res["c3_scan_i32"]["exchange"] = exchange.replace(
                "C3: scan pass 1", "C3: round totals all-gathered by the scan kernel")
    # DRAM bytes per launch measured by ncu --set full at the 1-GPU BASELINE
    # size (profiles/ncu_traffic.json) next to the algorithmic bytes
    if world == 1:
        for k, op in (("c1_reduce_i32", "reduce_sum_i32"), ("c3_scan_i32", "scan_inclusive_i32"),
                      ("c4_compact_i32", "compact_gt0_i32"), ("c5_hist_u8", "histogram256_u8")):
            if k in res:
                res[k]["ncu_dram_bytes"] = ncu_traffic(op)
                res[k]["algorithmic_bytes"] = int(res[k]["n"] * res[k]["bytes_per_elem"])
    del u
    torch.cuda.empty_cache()
    if world == 1:
        log("rank 0: reference formulations via launch(hybrid_transform(...))")
        res["via_reference_api"] = reference_api_rows(dev, peak, steps, warm, checks)
    return res


def warpfold_python_sample(n: int = 1 << 20) -> dict | None:
    """The reference's OWN CPU path, unmodified: warpfold's
    launch(hybrid_transform(kernel)) (runtime/launch.py:90,
    passes/pipeline.py:103) with all host cores as fork workers, from the
    copy installed in baseline/_ref, on the formulations SURVEY §8(d) names:
    the per-warp-partials reduction of §8c in fp32 (C2, the top-level
    fields) and int32 (C1), and the lane-reversed warp prefix (C3, warp
    level) — 2^20 elements each, results checked.  C4 / C5 have no reference
    path (not expressible in its DSL).  Supplementary: the arm's `value`
    stays the compiled restatement (orders of magnitude faster, so the
    conservative denominator)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "warpfold").is_dir():
        return {"unavailable": "baseline/_ref/warpfold not installed"}
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import numpy as np
        from warpfold import DeviceMemory, LaunchConfig, hybrid_transform, parse_module
        from warpfold.runtime.launch import launch
        from oracle import synthetic
        workers = os.cpu_count() or 1
        block = 256

        def timed(spk, gen, dtype, grid, out_len, with_n):
            kernel = parse_module((ROOT / "tests" / "golden" / spk).read_text()).kernel()
            cfg = LaunchConfig(grid_size=grid, block_size=block, warp_size=32, workers=workers)
            mem = DeviceMemory()
            a, out = mem.alloc(4 * n), mem.alloc(4 * out_len)
            x = synthetic.generate(gen, n, seed=1)
            mem.view(a, dtype)[:] = x
            prog = hybrid_transform(kernel, cfg)
            t = time.perf_counter()
            launch(prog, cfg, mem, [a, out, n] if with_n else [a, out])
            el = time.perf_counter() - t
            row = {"value": round(n / el / 1e9, 9), "unit": "Gelem/s", "cores": workers,
                   "kind": "reference", "sample": f"one launch over 2^{n.bit_length() - 1} {dtype} "
                   f"elements ({spk}), grid {grid} x block {block}, {workers} fork workers, "
                   f"{el:.2f} s"}
            return row, x, np.array(mem.view(out, dtype))

        grid = 8 * workers
        res, x, parts = timed("C1_F32.spk", "f32_unit", "f32", grid, grid * block // 32, True)
        total = np.float32(0)
        for v in parts:
            total = np.float32(total + v)
        res["result"] = float(total)
        rows = {"c2_reduce_f32": dict(res)}
        row, x, parts = timed("C1_I32.spk", "i32_full", "i32", grid, grid * block // 32, True)
        want = int(x.astype(np.int64).sum()) & 0xFFFFFFFF
        row["checked"] = (int(parts.astype(np.int64).sum()) & 0xFFFFFFFF) == want
        rows["c1_reduce_i32"] = row
        row, x, y = timed("C3_WARP_PREFIX.spk", "i32_full", "i32", n // block, n, False)
        w = x.astype(np.int64).reshape(-1, 32)
        want_p = np.cumsum(w, axis=1)  # per-warp inclusive prefix (lane-reversed suffix scan)
        row["checked"] = bool(np.array_equal(y.astype(np.int64).reshape(-1, 32) & 0xFFFFFFFF,
                                             want_p & 0xFFFFFFFF))
        rows["c3_warp_prefix_i32"] = row
        rows["c4_compact_i32"] = rows["c5_hist_u8"] = {
            "unavailable": "no reference path: not expressible in the reference DSL "
                           "(no ballot / atomics / u8, dsl/lexer.py:18-25, dsl/parser.py:83-88)"}
        res["per_kernel"] = rows
        return res
    except Exception as e:  # the supplementary leg never fails the arm
        return {"unavailable": f"{type(e).__name__}: {e}"}


def run_reference(args, rank, world) -> dict | None:
    """CPU arm: the collapsed-loop restatement of the reference on the host
    cores (rank 0 only); each step a bounded sample of the C2 workload."""
    if rank != 0:
        return None
    from oracle import cref
    cref.build()
    workers = cref.workers_default()
    pool = _cpu_c2_pool()
    # one step = one pass over the whole 2^27-element DRAM-resident pool
    # (8 slices, ~30-60 ms): long enough that thread start-up and clock ramp
    # do not understate the CPU (2^24-element steps measured 2.5 vs 4.4
    # Gelem/s for the same code in a 10 s run on the same box)
    slices = len(pool) >> CPU_SLICE_LOG2
    sample_n = slices << CPU_SLICE_LOG2
    grid = 64 * workers

    def step():
        for j in range(slices):
            _cpu_c2_run(pool, j, workers)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        step()
        times.append(time.perf_counter() - t)
    ms = statistics.mean(times) * 1e3
    value = sample_n / (ms * 1e-3) / 1e9
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gelem/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C2: fp32 warp-shuffle reduction over 2^30 elements "
                               f"(CPU: bounded 2^{CPU_POOL_LOG2}-element DRAM-resident sample per step)",
                   "n": N_C2, "block": 256, "parallelism": f"cpu{workers}"},
        "cpu_baseline": {"value": round(value, 6), "unit": "Gelem/s", "cores": workers,
                         "kind": "port",
                         "sample": f"one pass per step over a 2^{CPU_POOL_LOG2}-element "
                                   f"DRAM-resident fp32 pool ({slices} x 2^{CPU_SLICE_LOG2} slices), "
                                   f"through oracle/collapse_ref.c "
                                   f"(per-warp-partials shfl_down kernel collapsed into "
                                   f"block/warp/lane loops, grid {grid} x 256, {workers} threads)"},
        "e2e": {"value": round(value, 6), "unit": "Gelem/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "warpfold_python": None if args.no_cpu_baseline else warpfold_python_sample(),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-shards", action="store_true",
                    help="skip the one-GPU scaling prediction (predicted_scaling)")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        # not launched by torchrun: become the launcher (one rank per GPU)
        sys.exit(relaunch_under_torchrun(args.gpus))
    if int(env_world or "1") != args.gpus:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}: refusing to measure "
            f"a different GPU count than requested")
        sys.exit(2)
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    rank, world, local = init_dist(args)
    line = run_ours(args, rank, world, local)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if line is not None and not all(line["verified"].values()):
        log(f"bench.py: result check FAILED: {line['verified']}")
        sys.exit(3)


def relaunch_under_torchrun(n: int) -> int:
    """`python bench.py --gpus N` without torchrun: re-exec this command as
    N ranks (`torch.distributed.run --nproc-per-node N`, 127.0.0.1)."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(Path(__file__).resolve()), *sys.argv[1:]]
    log("bench.py: relaunching as " + " ".join(cmd[1:]))
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()
