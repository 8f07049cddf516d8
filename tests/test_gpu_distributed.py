"""The N>1 combine path on real kernels, one GPU.

The GPU runs of this project are single-GPU, so NCCL with world_size > 1
cannot run here.  These tests drive `paper_2112_10034_b200.distributed` as
rank r of a world of W with the collective replaced by its exact result (the
stacked per-rank values that an all-gather / all-reduce would deliver, computed
by the same sm_100a kernels on the other ranks' shards).  What is under test
is everything the product does around the collective on the device: the
fixed-order fold of partials (bit-identical on every rank), the exclusive
carry fed to the scan, the global compaction offsets and the bin sums —
checked against the oracle over the whole (unsharded) input."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import numpy_oracle as no, synthetic  # noqa: E402


@pytest.fixture(scope="module")
def wd():
    from paper_2112_10034_b200 import build
    build.build_library()
    from paper_2112_10034_b200 import distributed
    torch.cuda.init()
    return distributed


def _as_rank(monkeypatch, wd, rank, world, gathered):
    """Make `wd` believe it is rank `rank` of `world`; all-gathers return the
    per-rank values in `gathered[dtype]`, all-reduces sum `gathered['bins']`."""
    monkeypatch.setattr(wd, "_world", lambda group=None: (rank, world))

    def exchange(local, group=None):
        rows = gathered[local.dtype]
        assert torch.equal(rows[rank].reshape(local.shape), local), "local value differs"
        return torch.stack([r.reshape(local.shape) for r in rows])

    def all_reduce(t, op=None, group=None):
        t.copy_(torch.stack(gathered["bins"]).sum(0))

    monkeypatch.setattr(wd, "exchange", exchange)
    monkeypatch.setattr(wd.dist, "all_reduce", all_reduce)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_reductions_scan_compaction(wd, monkeypatch, world):
    from paper_2112_10034_b200 import ops
    n = 5 * 8192 * world + 4099  # ragged: the last shard is short
    shards = [wd.shard_range(n, r, world) for r in range(world)]
    xf = [ops.fill_synthetic("f32_unit", hi - lo, seed=4, base=lo) for lo, hi in shards]
    xi = [ops.fill_synthetic("i32_full", hi - lo, seed=5, base=lo) for lo, hi in shards]
    gathered = {
        torch.float32: [ops.reduce_sum_f32(x) for x in xf],
        torch.int32: [ops.reduce_sum_i32(x) for x in xi],
        torch.int64: [ops.compact_gt0_i32(x)[1] for x in xi],
    }
    whole_i = synthetic.generate("i32_full", n, seed=5)
    whole_f = synthetic.generate("f32_unit", n, seed=4)
    f32_bits, i32_vals, scan_parts, comp_parts = set(), set(), [], []
    for r in range(world):
        _as_rank(monkeypatch, wd, r, world, gathered)
        f32_bits.add(int(wd.reduce_sum_f32(xf[r]).view(torch.int32).item()))
        i32_vals.add(int(wd.reduce_sum_i32(xi[r]).item()))
        scan_parts.append(wd.scan_inclusive_i32(xi[r]).cpu().numpy())
        out, cnt, off, tot = wd.compact_gt0_i32(xi[r])
        m = int(cnt.item())
        comp_parts.append((int(off.item()), out[:m].cpu().numpy(), int(tot.item())))
    assert len(f32_bits) == 1, "fp32 fold must be bit-identical on every rank"
    got = np.array([f32_bits.pop()], dtype=np.int32).view(np.float32)[0]
    assert abs(float(got) - no.reduce_sum_f32_exact(whole_f)) <= no.f32_tolerance(n, no.abs_sum(whole_f))
    assert i32_vals == {int(no.reduce_sum_i32(whole_i))}
    assert np.array_equal(np.concatenate(scan_parts), no.scan_inclusive_i32(whole_i))
    want = no.compact_gt0_i32(whole_i)
    pos = 0
    for off, part, tot in comp_parts:
        assert off == pos and tot == len(want)
        assert np.array_equal(part, want[pos:pos + len(part)])
        pos += len(part)
    assert pos == len(want)


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_histogram(wd, monkeypatch, world):
    from paper_2112_10034_b200 import ops
    n = 3 * 4096 * world + 77
    shards = [wd.shard_range(n, r, world) for r in range(world)]
    xs = [ops.fill_synthetic("u8_uniform", hi - lo, seed=6, base=lo) for lo, hi in shards]
    gathered = {"bins": [ops.histogram256_u8(x).clone() for x in xs]}
    want = no.histogram256_u8(synthetic.generate("u8_uniform", n, seed=6))
    for r in range(world):
        _as_rank(monkeypatch, wd, r, world, gathered)
        got = wd.histogram256_u8(xs[r]).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want)


@pytest.mark.slow
def test_bench_n2_path_simulated(wd, monkeypatch):
    """bench.py's N>1 code path (rank 0 of 2) end to end on one GPU: the
    collectives return what a peer holding identical values would deliver.
    Catches host-side errors in the sharded bench legs the driver's scaling
    run would take; the numbers are not a measurement."""
    import argparse
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    import torch.distributed as dist

    monkeypatch.setattr(wd, "_world", lambda group=None: (0, 2))
    monkeypatch.setattr(wd, "exchange", lambda local, group=None:
                        torch.stack([local.reshape(local.shape)] * 2))
    monkeypatch.setattr(dist, "barrier", lambda *a, **k: None)
    monkeypatch.setattr(dist, "all_reduce", lambda t, *a, **k: t)
    args = argparse.Namespace(gpus=2, steps=3, warmup=3, impl="ours", headline_only=False,
                              no_cpu_baseline=True, cpu_budget=1.0)
    line = bench.run_ours(args, 0, 2, 0)
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "shard2"
    assert line["gpu_launches"] == 2 * args.steps  # K2 + fold per step
    per = line["per_kernel"]
    assert per["c3_scan_i32"]["bytes_per_elem"] == 12  # reduce-then-scan across GPUs
    for k in ("c1_reduce_i32", "c3_scan_i32", "c4_compact_i32", "c5_hist_u8"):
        assert per[k]["gelem_s"] > 0


@pytest.mark.slow
@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_bench_cyclic_scan_processes_one_gpu(nproc):
    """bench.py at N = 2 / 4 / 8 with C3 on the block-cyclic single-pass
    scan, as real processes (torchrun, gloo, IPC mailboxes) time-slicing GPU
    0: the kernels wait on each other's round totals mid-kernel across
    contexts; every leg's result is checked (the C3 check regenerates the
    global array and compares every super-tile).  The driver's 8-GPU
    scaling run takes this code path with one GPU per rank."""
    import json
    import os
    import socket
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, WF_BENCH_SAME_GPU="1", WF_BENCH_BACKEND="gloo", WF_BENCH_CYCLIC="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", str(nproc), "--master-addr", "127.0.0.1",
                        "--master-port", str(port), "bench.py", "--gpus", str(nproc),
                        "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-shards"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == nproc and line["config"]["parallelism"] == f"shard{nproc}"
    c3 = line["per_kernel"]["c3_scan_i32"]
    assert c3["layout"].startswith("block-cyclic") and c3["bytes_per_elem"] == 8
    assert line["verified"]["c3_scan_i32"] is True
    assert all(line["verified"].values()), line["verified"]
    for k in ("c3_scan_i32", "c4_compact_i32", "c5_hist_u8"):
        assert "FAILED" not in line["per_kernel"][k]["exchange"], line["per_kernel"][k]


@pytest.mark.slow
def test_bench_n2_two_processes_one_gpu():
    """bench.py at N=2 as the driver launches it (torchrun, one process per
    rank), with both ranks on GPU 0 over gloo (WF_BENCH_SAME_GPU): real
    process group, IPC mailboxes and fused exchanges, so a collective issued
    by only some ranks (it once hung the C1 leg's stats) or a mismatched
    epoch sequence fails here.  Numbers are meaningless (two contexts
    time-slice one GPU); only completion and the line's shape are checked."""
    import json
    import os
    import socket
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, WF_BENCH_SAME_GPU="1", WF_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "shard2"
    assert line["config"]["exchange"].startswith("peer memory"), line["config"]["exchange"]
    assert line["gpu_launches"] == line["steps"]  # one fused kernel per step
    for k in ("c3_scan_i32", "c4_compact_i32", "c5_hist_u8"):
        assert "FAILED" not in line["per_kernel"][k]["exchange"], line["per_kernel"][k]
    assert "FAILED" not in line["config"]["exchange"]
