"""The GPU mode-comparison bench (`python -m paper_2112_10034_b200 bench`,
the reference's cli.py:128-151 / bench.py:53-126 analogue)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

from paper_2112_10034_b200 import benchmarks as bm
from paper_2112_10034_b200.__main__ import build_parser
from paper_2112_10034_b200.config import LaunchConfig
from paper_2112_10034_b200.dsl import hybrid_transform, specialize

ROOT = Path(__file__).resolve().parents[1]


def test_parser_accepts_reference_bench_flags():
    a = build_parser().parse_args(["bench", "--suite", "modes", "--iters", "10",
                                   "--repeats", "2", "--json"])
    assert (a.suite, a.iters, a.repeats, a.json) == ("modes", 10, 2, True)


@pytest.mark.parametrize("name", bm.MODE_KERNELS)
def test_mode_kernels_translate_both_ways(name):
    k = bm._kernel(bm.MODE_SOURCES[name])
    cfg = LaunchConfig(grid_size=1, block_size=32)
    for mode in ("flat", "hier"):
        assert "__global__" in hybrid_transform(k, cfg, mode=mode).cuda_source(cfg)


def test_jit_kernel_specializes():
    cfg = LaunchConfig(grid_size=1, block_size=32)
    prog = specialize(hybrid_transform(bm._kernel(bm.JIT_SOURCE), cfg, mode="hier"), cfg)
    assert prog.specialized == {"block_size": 32, "grid_size": 1}


@pytest.mark.gpu
def test_bench_cli_all_suites():
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    r = subprocess.run([sys.executable, "-m", "paper_2112_10034_b200", "bench", "--json",
                        "--iters", "20", "--repeats", "2", "--op-iters", "3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert [row["kernel"] for row in res["modes"]] == list(bm.MODE_KERNELS)
    assert all(row["flat_ms"] > 0 and row["hier_ms"] > 0 for row in res["modes"])
    assert res["jit"]["specialized_ms"] > 0
    assert len(res["ops"]) == sum(len(v[2]) for v in bm.OPS.values())
    assert all(row["gelem_s"] > 0 for row in res["ops"])
    assert [row["n_gpus"] for row in res["scaling"]] == [1] * 4
    assert [(row["op"], row["n_gpus"]) for row in res["shards"]][:4] == [
        ("reduce_sum_f32", 1), ("reduce_sum_f32", 2), ("reduce_sum_f32", 4), ("reduce_sum_f32", 8)]
    assert all(row["per_rank_us"] > 0 for row in res["shards"])


@pytest.mark.gpu
def test_bench_shards_small_totals():
    """The one-GPU scaling prediction at small totals: every op at 1/2/4
    shards, per-rank steps shrink with the shard, speed-ups are relative to
    the 1-shard step."""
    import torch
    rows = bm.bench_shards(worlds=(1, 2, 4), iters=3, repeats=2,
                           log2_total={"reduce_sum_f32": 24, "scan_inclusive_i32": 22,
                                       "compact_gt0_i32": 22, "histogram256_u8": 26})
    assert len(rows) == 12 and torch.cuda.is_available()
    for r in rows:
        assert r["per_rank_us"] > 0
        if r["n_gpus"] == 1:
            assert r["predicted_speedup"] == 1.0


@pytest.mark.gpu
@pytest.mark.slow
def test_bench_cli_scaling_two_processes_one_gpu():
    """`bench --suite scaling` under torchrun with 2 ranks (both on GPU 0
    over gloo, WF_BENCH_SAME_GPU): the fused peer exchanges are set up by
    consensus and every rank issues the same collectives."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, PYTHONPATH=str(ROOT), WF_BENCH_SAME_GPU="1", WF_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), "-m", "paper_2112_10034_b200", "bench",
                        "--suite", "scaling", "--json", "--op-iters", "3", "--repeats", "2"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    rows = json.loads(r.stdout.strip().splitlines()[-1])["scaling"]
    assert [row["n_gpus"] for row in rows] == [2] * 4
    assert all(row["exchange"] == "peer memory (fused)" for row in rows), rows


def test_bench_refuses_a_world_size_other_than_gpus():
    """`--gpus N` is the GPU count measured: under a launcher whose world size
    differs, bench.py exits non-zero instead of reporting another N."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference",
                        "--no-cpu-baseline"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 2 and "refusing" in r.stderr
