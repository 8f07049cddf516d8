"""GPU counterpart of the reference's mode-comparison harness
(warpfold/bench.py:53-126, CLI ``bench`` at cli.py:128-151, :201-206).

The reference times translation modes on CPU workers: flat vs hierarchical
lane loops (``bench_modes``), normal vs configuration-folded programs
(``bench_jit``) and a worker sweep (``bench_scaling``).  On the B200 the same
three questions become

  modes    flat vs hier translation of barrier-free DSL kernels, compiled to
           sm_100a and launched through ``runtime.launch`` (join semantics:
           wall time per launch including the synchronise, as the reference
           times launch + join).  There are no lane loops on the GPU, so the
           ratio is ~1 — the direction the reference asserts (hier >= flat)
           collapses to parity.
  jit      normal vs ``specialize``d (blockDim/gridDim folded into the NVRTC
           source) for the C1 pin kernel.
  ops      the five warp-primitive kernels (K1-K5) over a size sweep: device
           time by CUDA events, Gelem/s and algorithmic GB/s.
  scaling  the sharded K2-K5 (``distributed.py``) at a fixed total size on
           every rank of the process group (launch under torchrun for
           1/2/4/8 GPUs): device time, max over ranks — the 1/2/4/8-GPU
           curve that replaces the reference's worker sweep.
  shards   the same curve predicted on ONE GPU: the per-rank step of each
           sharded op at the 1/2/4/8-GPU shard sizes, run with the fused
           kernels on a world-1 mailbox (the exchange protocol executes; the
           NVLink round trip, ~1-2 us, does not), steps as dependent
           launches; speed-up = t(1 GPU) / t(N)  (bench_shards).

All inputs are synthetic (``ops.fill_synthetic``) and generated in HBM.
"""

from __future__ import annotations

import statistics
import time

import torch

from . import ops
from .config import LaunchConfig
from .memory import DeviceMemory

NOMINAL_HBM_GBS = 8000.0  # north_star's 8 TB/s
C3_ROUND = 1 << 22        # block-cyclic super-tile of the sharded scan (bench.py C3_ROUND)
L2_BYTES = 126 << 20      # B200 L2: inputs at or below this stay resident across repeats

# Barrier-free kernels for the modes suite (the reference uses the same four
# names, bench.py:24); written here for the GPU bench.
MODE_SOURCES = {
    "veccopy": """
__global__ void veccopy(global i32* a, global i32* b) {
    i32 i = threadIdx.x + blockIdx.x * blockDim.x;
    b[i] = a[i];
}""",
    "vecadd": """
__global__ void vecadd(global i32* a, global i32* b, global i32* c) {
    i32 i = threadIdx.x + blockIdx.x * blockDim.x;
    c[i] = a[i] + b[i];
}""",
    "saxpy": """
__global__ void saxpy(global f32* x, global f32* y, f32 alpha) {
    i32 i = threadIdx.x + blockIdx.x * blockDim.x;
    y[i] = alpha * x[i] + y[i];
}""",
    "matmul": """
__global__ void matmul(global f32* a, global f32* b, global f32* c, i32 k) {
    i32 row = blockIdx.x;
    i32 col = threadIdx.x;
    f32 acc = 0.0;
    for (i32 j = 0; j < k; j = j + 1) {
        acc = acc + a[row * k + j] * b[j * blockDim.x + col];
    }
    c[row * blockDim.x + col] = acc;
}""",
}
MODE_KERNELS = tuple(MODE_SOURCES)

# The C1 pin kernel: grid-stride sum, five shfl_down rounds,
# one partial per warp.
JIT_SOURCE = """
__global__ void wsum(global i32* a, global i32* out, i32 n) {
    i32 tx = threadIdx.x;
    i32 sum = 0;
    for (i32 i = tx + blockIdx.x * blockDim.x; i < n; i = i + blockDim.x * gridDim.x) {
        sum = sum + a[i];
    }
    for (i32 off = 16; off > 0; off = off / 2) {
        sum = sum + shfl_down(sum, off);
    }
    if (tx % 32 == 0) {
        out[blockIdx.x * (blockDim.x / 32) + tx / 32] = sum;
    }
}"""

# (op, generator, algorithmic bytes per element, default log2 sizes)
OPS = {
    "reduce_sum_i32": ("i32_full", 4.0, (20, 24, 28)),
    "reduce_sum_f32": ("f32_unit", 4.0, (24, 28, 30)),
    "scan_inclusive_i32": ("i32_full", 8.0, (20, 24, 28)),
    "compact_gt0_i32": ("i32_full", None, (20, 24, 28)),  # 4 + 4*selected/n
    "histogram256_u8": ("u8_uniform", 1.0, (24, 28, 32)),
}


def _kernel(source: str):
    from .dsl import parse_module
    return parse_module(source).kernel(None)


def time_launches(program, config, memory, args, iters: int) -> float:
    """Total wall seconds for `iters` launches (each one joins, like the
    reference's time_launches, bench.py:27-31)."""
    from .runtime import launch
    t0 = time.perf_counter()
    for _ in range(iters):
        launch(program, config, memory, args)
    return time.perf_counter() - t0


def _median_pair(a, b, iters: int, repeats: int) -> tuple[float, float]:
    """Interleaved timing of two setups (bench.py:40-50)."""
    from .runtime import launch
    for setup in (a, b):
        launch(*setup)
    ta, tb = [], []
    for _ in range(repeats):
        ta.append(time_launches(*a, iters))
        tb.append(time_launches(*b, iters))
    return statistics.median(ta), statistics.median(tb)


def _mode_setup(name: str, grid: int, block: int, mem: DeviceMemory):
    n = grid * block
    g = torch.Generator().manual_seed(7)
    if name in ("veccopy", "vecadd"):
        bufs = [mem.alloc(4 * n) for _ in range(2 if name == "veccopy" else 3)]
        for b in bufs:
            mem.copy_in(b, torch.randint(-100, 100, (n,), generator=g, dtype=torch.int32).numpy())
        return bufs
    if name == "saxpy":
        x, y = mem.alloc(4 * n), mem.alloc(4 * n)
        mem.copy_in(x, torch.randn(n, generator=g).numpy())
        mem.copy_in(y, torch.randn(n, generator=g).numpy())
        return [x, y, 2.0]
    k = 64
    a, b, c = mem.alloc(4 * grid * k), mem.alloc(4 * k * block), mem.alloc(4 * n)
    mem.copy_in(a, torch.randn(grid * k, generator=g).numpy())
    mem.copy_in(b, torch.randn(k * block, generator=g).numpy())
    return [a, b, c, k]


def bench_modes(kernels=MODE_KERNELS, iters: int = 1000, repeats: int = 5,
                grid: int = 1, block: int = 32, device=None) -> list[dict]:
    """Flat vs hierarchical translation on barrier-free kernels (bench.py:53-74)."""
    from .dsl import hybrid_transform
    rows = []
    for name in kernels:
        kernel = _kernel(MODE_SOURCES[name])
        mem = DeviceMemory(device)
        args = _mode_setup(name, grid, block, mem)
        cfg = LaunchConfig(grid_size=grid, block_size=block)
        flat = hybrid_transform(kernel, cfg, mode="flat")
        hier = hybrid_transform(kernel, cfg, mode="hier")
        fs, hs = _median_pair((flat, cfg, mem, args), (hier, cfg, mem, args), iters, repeats)
        rows.append({"kernel": name, "iters": iters, "grid": grid, "block": block,
                     "flat_ms": fs / iters * 1e3, "hier_ms": hs / iters * 1e3,
                     "hier_over_flat": hs / fs if fs else float("nan")})
    return rows


def bench_jit(iters: int = 1000, repeats: int = 5, grid: int = 1, block: int = 32,
              device=None) -> dict:
    """Normal vs configuration-folded program (bench.py:77-94)."""
    from .dsl import hybrid_transform, specialize
    kernel = _kernel(JIT_SOURCE)
    cfg = LaunchConfig(grid_size=grid, block_size=block)
    mem = DeviceMemory(device)
    n = grid * block * 4
    a, out = mem.alloc(4 * n), mem.alloc(4 * grid * max(1, block // 32))
    mem.copy_in(a, torch.randint(-10, 10, (n,), dtype=torch.int32).numpy())
    normal = hybrid_transform(kernel, cfg, mode="hier")
    folded = specialize(normal, cfg)
    ns, fs = _median_pair((normal, cfg, mem, [a, out, n]), (folded, cfg, mem, [a, out, n]),
                          iters, repeats)
    return {"kernel": "wsum", "iters": iters, "grid": grid, "block": block,
            "normal_ms": ns / iters * 1e3, "specialized_ms": fs / iters * 1e3,
            "specialized_over_normal": fs / ns if ns else float("nan")}


def _run_op(op: str, x: torch.Tensor, outs: dict):
    if op == "reduce_sum_i32":
        return ops.reduce_sum_i32(x, outs.get("out"))
    if op == "reduce_sum_f32":
        return ops.reduce_sum_f32(x, outs.get("out"), block=512)
    if op == "scan_inclusive_i32":
        return ops.scan_inclusive_i32(x, outs.get("out"))
    if op == "compact_gt0_i32":
        return ops.compact_gt0_i32(x, outs.get("out"), outs.get("count"))
    return ops.histogram256_u8(x, outs.get("bins"))


def _outs(op: str, n: int, device) -> dict:
    if op in ("reduce_sum_i32", "reduce_sum_f32"):
        dt = torch.int32 if op.endswith("i32") else torch.float32
        return {"out": torch.empty(1, dtype=dt, device=device)}
    if op == "scan_inclusive_i32":
        return {"out": torch.empty(n, dtype=torch.int32, device=device)}
    if op == "compact_gt0_i32":
        return {"out": torch.empty(n, dtype=torch.int32, device=device),
                "count": torch.empty(1, dtype=torch.int64, device=device)}
    return {"bins": torch.empty(256, dtype=torch.int64, device=device)}


def _device_time(fn, iters: int, repeats: int) -> float:
    """Median over `repeats` of (CUDA-event time of `iters` back-to-back
    calls) / iters, in seconds."""
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3 / iters)
    return statistics.median(ts)


def _bytes_per_elem(op: str, x: torch.Tensor, outs: dict) -> float:
    bpe = OPS[op][1]
    if bpe is None:  # compaction: read + selected writes
        return 4.0 + 4.0 * int(outs["count"].item()) / max(1, x.numel())
    return bpe


def bench_ops(ops_=tuple(OPS), log2_sizes=None, iters: int = 20, repeats: int = 5,
              device=None) -> list[dict]:
    """K1-K5 over a size sweep, device-timed."""
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    rows = []
    for op in ops_:
        gen, _, sizes = OPS[op]
        for lg in (log2_sizes or sizes):
            n = 1 << lg
            x = ops.fill_synthetic(gen, n, seed=0, device=device)
            outs = _outs(op, n, device)
            t = _device_time(lambda: _run_op(op, x, outs), iters, repeats)
            bpe = _bytes_per_elem(op, x, outs)
            gbs = n * bpe / t / 1e9
            rows.append({"op": op, "n": n, "us": t * 1e6, "gelem_s": n / t / 1e9,
                         "gbs": gbs, "frac_of_8tbs": gbs / NOMINAL_HBM_GBS,
                         "bytes_per_elem": bpe,
                         "l2_resident": x.numel() * x.element_size() <= L2_BYTES})
            del x, outs
    torch.cuda.empty_cache()
    return rows


def bench_scaling(ops_=("reduce_sum_f32", "scan_inclusive_i32", "compact_gt0_i32",
                        "histogram256_u8"), log2_total=None, iters: int = 20,
                  repeats: int = 5, group=None, peer: bool = True) -> list[dict]:
    """Sharded K2-K5 at a fixed total size (strong scaling) on every rank of
    the process group; time = max over ranks of the device time.  With
    `peer` the exchanges run fused into the kernels over peer memory
    (p2p.PeerReducer / PeerCollectives, set up by consensus; NCCL if any rank
    cannot map the others' mailboxes).  Without a process group it measures
    one GPU."""
    import torch.distributed as dist
    from . import distributed as wd
    dev = torch.device("cuda", torch.cuda.current_device())
    rank, world = (dist.get_rank(group), dist.get_world_size(group)) \
        if dist.is_available() and dist.is_initialized() else (0, 1)
    totals = log2_total or {"reduce_sum_f32": 30, "scan_inclusive_i32": 28,
                            "compact_gt0_i32": 28, "histogram256_u8": 32}
    pr = pc = None
    exchange = "none (1 GPU)"
    if world > 1:
        exchange = "NCCL"
        if peer:
            from . import p2p
            lo_p, hi_p = wd.shard_range(1 << 20, rank, world)
            probe = ops.fill_synthetic("f32_unit", hi_p - lo_p, seed=7, base=lo_p, device=dev)
            pr, _ = p2p.try_peer_reducer(dev, probe, group)
            pc, _ = p2p.try_peer_collectives(dev, group)
            exchange = "peer memory (fused)" if pr is not None and pc is not None else "NCCL"
            if exchange == "NCCL":  # identical decision on every rank (consensus above)
                pr = pc = None
    rows = []
    for op in ops_:
        gen = OPS[op][0]
        n = 1 << totals[op]
        lo, hi = wd.shard_range(n, rank, world)
        layout = "contiguous"
        if op == "scan_inclusive_i32" and pc is not None:
            # block-cyclic super-tiles, single-pass scan (as bench.py at N > 1)
            rounds, parts = wd.cyclic_rounds(n, rank, world, C3_ROUND)
            x = torch.empty(sum(m for _, m in parts), dtype=torch.int32, device=dev)
            off = 0
            for start, m in parts:
                ops.fill_synthetic(gen, m, seed=0, base=start, out=x[off:off + m])
                off += m
            layout = f"block-cyclic ({C3_ROUND}-element super-tiles)"
        else:
            x = ops.fill_synthetic(gen, hi - lo, seed=0, base=lo, device=dev)
        outs = _outs(op, x.numel(), dev)
        if op == "reduce_sum_f32":
            fn = (lambda: pr.reduce_sum_f32(x, block=512)) if pr is not None else \
                (lambda: wd.reduce_sum_f32(x, group=group, block=512))
        elif op == "scan_inclusive_i32" and pc is not None:
            fn = lambda: pc.scan_inclusive_i32_cyclic(x, outs["out"], C3_ROUND,  # noqa: E731
                                                      rounds)
        elif op == "scan_inclusive_i32":
            fn = lambda: wd.scan_inclusive_i32(x, outs["out"], group=group, peer=pc)  # noqa: E731
        elif op == "compact_gt0_i32":
            fn = lambda: wd.compact_gt0_i32(x, outs["out"], group=group, peer=pc)  # noqa: E731
        else:
            fn = lambda: wd.histogram256_u8(x, group=group, peer=pc)  # noqa: E731
        if world > 1:
            dist.barrier(group=group)
        t = torch.tensor([_device_time(fn, iters, repeats)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        t = float(t.item())
        rows.append({"op": op, "n": n, "n_gpus": world, "scaling": "strong",
                     "us": t * 1e6, "gelem_s": n / t / 1e9, "exchange": exchange,
                     "layout": layout})
        del x, outs
    failed = pc is not None and pc.failed()
    for closer in (pr, pc):
        if closer is not None:
            torch.cuda.synchronize()
            closer.close()
    if failed:
        for r in rows:
            r["exchange"] += " — FAILED (peer timeout)"
    torch.cuda.empty_cache()
    return rows


def bench_shards(worlds=(1, 2, 4, 8), log2_total=None, iters: int = 20, repeats: int = 5,
                 device=None) -> list[dict]:
    """Predicted strong scaling on one GPU (module docstring, `shards`).  At
    N = 1 the single-GPU ops run (what bench.py times at 1 GPU); at N > 1 the
    fused per-rank kernels bench.py runs on each rank (p2p.PeerReducer /
    PeerCollectives), here on a world-1 mailbox.  Every step is a
    WF_FLAG_INPUT_STABLE launch, as in bench.py; each op's shard sizes are
    interleaved round by round."""
    from . import p2p
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    totals = log2_total or {"reduce_sum_f32": 30, "scan_inclusive_i32": 28,
                            "compact_gt0_i32": 28, "histogram256_u8": 32}
    boxes = p2p.Mailboxes.local(1, dev, cap=256)
    kboxes = p2p.Mailboxes.local(1, dev)
    pc = p2p.PeerCollectives(boxes[0], 0, 1, 256, dev)
    pr = p2p.PeerReducer(kboxes[0], 0, 1)
    step_us: dict = {}

    def step_fn(op, world, x, y):
        if op == "reduce_sum_f32":
            red = ops.reduce_sum_f32 if world == 1 else pr.reduce_sum_f32
            return lambda: red(x, block=256, input_stable=True)
        if op == "scan_inclusive_i32":
            if world == 1:
                return lambda: ops.scan_inclusive_i32(x, y, input_stable=True)
            # bench.py's N > 1 path: block-cyclic super-tiles, single pass
            rounds = -(-x.numel() // C3_ROUND)
            return lambda: pc.scan_inclusive_i32_cyclic(x, y, C3_ROUND, rounds,
                                                        input_stable=True)
        if op == "compact_gt0_i32":
            if world == 1:
                return lambda: ops.compact_gt0_i32(x, y, input_stable=True)
            return lambda: pc.compact_gt0_i32(x, y, input_stable=True)
        if world == 1:
            return lambda: ops.histogram256_u8(x, input_stable=True)
        return lambda: pc.histogram256_u8(x, input_stable=True)

    try:
        # one op at a time, its shard sizes interleaved round by round: every
        # timed loop follows the same op (no other op's dirty L2 lines), and
        # clock / power drift hits every N alike
        for op in totals:
            fns = {}
            for world in worlds:
                x = ops.fill_synthetic(OPS[op][0], (1 << totals[op]) // world, seed=0, device=dev)
                y = torch.empty(x.numel(), dtype=torch.int32, device=dev) \
                    if op in ("scan_inclusive_i32", "compact_gt0_i32") else None
                fns[world] = step_fn(op, world, x, y)
            times = {world: [] for world in worlds}
            torch.cuda.synchronize()  # the fills above wrote the inputs
            for fn in fns.values():
                fn()
            for _ in range(repeats):
                for world, fn in fns.items():
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(iters):
                        fn()
                    e1.record()
                    e1.synchronize()
                    times[world].append(e0.elapsed_time(e1) * 1e3 / iters)
            for world, v in times.items():
                step_us[(op, world)] = statistics.median(v)
            del fns
            torch.cuda.empty_cache()
        if pc.failed():
            raise RuntimeError("bench_shards: the fused exchange timed out")
    finally:
        torch.cuda.synchronize()
        boxes[0].close()
        kboxes[0].close()
    rows = []
    for op in totals:
        t1 = step_us.get((op, worlds[0]))
        for world in worlds:
            t = step_us[(op, world)]
            rows.append({"op": op, "n": 1 << totals[op], "n_gpus": world, "scaling": "strong",
                         "per_rank_us": t, "predicted_speedup": t1 / t * worlds[0],
                         "predicted_efficiency": t1 / t * worlds[0] / world,
                         "how": "one GPU: per-rank step at this shard size, world-1 fused "
                                "protocol (NVLink round trip not included)"})
    torch.cuda.empty_cache()
    return rows

