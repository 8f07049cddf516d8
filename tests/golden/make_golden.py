"""Generate golden vectors by running the warpfold reference itself.

Run in the container that has the read-only reference mounted:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes small fixtures next to this script.  The GPU box never reads the
reference: tests load only these committed files.  Every vector comes from
the reference's own code paths:
  - warp_semantics.json: passes/warp_lower.py shuffle_down / reduce_vote
  - oracle_kat.npz: interp/oracle.py run_oracle on the kernels of the
    reference's tests/test_oracle.py:41-89 known-answer tests
  - c1c2_pin.npz: the SURVEY.md §8c per-warp-partials shfl_down reduction
    (i32 and f32) through BOTH run_oracle and launch(hybrid_transform(...))
  - c3_pin.npz: warp inclusive prefix scan (lane-reversed shfl_down, the only
    formulation the reference DSL can express) through run_oracle and launch
  - c4c5_pin.npz: ordered stream compaction (x > 0) and the 256-bin byte
    histogram.  The reference DSL has no ballot, atomics or u8
    (dsl/lexer.py:18-25, dsl/parser.py:83-88), so the warp-aggregated /
    smem-privatised algorithms are not expressible; these are the semantic
    formulations it CAN express (a serial in-order compaction thread; one
    thread per bin counting i32-widened bytes), run through run_oracle and
    launch(hybrid_transform(...)) — reference-produced vectors that pin the
    results K4 / K5 must reproduce
  - random_kernels.json: 200 kernels from the reference's own fuzzer
    (randgen.generate_kernel, the inputs of tests/test_random_diff.py:17-27)
    with their run_oracle outputs — cross-checked against the transformed
    path, as the reference's differential test does
  - acceptance_fuzz.json: the 1000 fuzzer kernels of the reference's
    acceptance criterion 5 with their run_oracle outputs
  - corpus.npz: all 17 corpus kernels (corpus.py) through run_oracle
  - corpus_traces.json: run_oracle ExecTrace counts for the same runs and the
    cfg/build.py uid -> IR-class catalogue of every kernel (--traces-only
    regenerates just this file)
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))  # repo root, for oracle.synthetic

from warpfold import DeviceMemory, LaunchConfig, hybrid_transform, parse_module, run_oracle  # noqa: E402
from warpfold import corpus  # noqa: E402
from warpfold.passes.warp_lower import reduce_vote, shuffle_down  # noqa: E402
from warpfold.runtime.launch import bind_args, launch  # noqa: E402

from oracle import synthetic  # noqa: E402

C1_I32 = """
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
}
"""
C1_F32 = C1_I32.replace("global i32* a, global i32* out", "global f32* a, global f32* out") \
               .replace("i32 sum = 0;", "f32 sum = 0.0;")

C3_WARP_PREFIX = """
__global__ void warp_prefix(global i32* a, global i32* out) {
    i32 tid = threadIdx.x + blockIdx.x * blockDim.x;
    i32 lane = threadIdx.x % 32;
    i32 base = tid - lane;
    i32 v = a[base + 31 - lane];
    for (i32 off = 1; off < 32; off = off * 2) {
        i32 t = shfl_down(v, off);
        if (lane + off < 32) {
            v = v + t;
        }
    }
    out[base + 31 - lane] = v;
}
"""


def _run(engine: str, source: str, grid: int, block: int, buffers, scalars=(), warp=32):
    kernel = parse_module(source).kernel()
    cfg = LaunchConfig(grid_size=grid, block_size=block, warp_size=warp, workers=1)
    mem = DeviceMemory()
    args = []
    for kind, init in buffers:
        buf = mem.alloc(4 * len(init))
        mem.view(buf, kind)[:] = init
        args.append(buf)
    args.extend(scalars)
    if engine == "oracle":
        run_oracle(kernel, cfg, bind_args(kernel.params, mem, args))
    else:
        cfg.workers = 8
        launch(hybrid_transform(kernel, cfg), cfg, mem, args)
    return [mem.view(b, kind).copy() for (kind, _), b in zip(buffers, args)]


def warp_semantics() -> dict:
    lanes = list(range(100, 132))
    table = [[int(shuffle_down(lanes, lane, off, 32)) for off in range(-40, 40)]
             for lane in range(32)]
    votes = {}
    for width in (4, 8):
        rows = []
        for m in range(1 << width):
            bits = [(m >> k) & 1 for k in range(width)]
            rows.append([m, reduce_vote(bits, "all"), reduce_vote(bits, "any")])
        votes[str(width)] = rows
    return {"source": "warpfold passes/warp_lower.py:17-45",
            "shfl_down": {"buffer": lanes, "offsets": list(range(-40, 40)), "table": table},
            "reduce_vote": votes}


def oracle_kat() -> dict:
    reduce_src = """
__global__ void reduce_warp(global i32* a, global i32* out) {
    i32 tid = threadIdx.x + blockIdx.x * blockDim.x;
    i32 val = a[tid];
    if (threadIdx.x < 32) {
        for (i32 offset = 16; offset > 0; offset = offset / 2) {
            val = val + shfl_down(val, offset);
        }
    }
    if (threadIdx.x == 0) { out[blockIdx.x] = val; }
    a[tid] = val;
}
"""
    out = {}
    a, o = _run("oracle", reduce_src, 1, 64, [("i32", np.ones(64)), ("i32", np.zeros(1))])
    out["kat_ones_a"], out["kat_ones_out"] = a, o
    data = np.arange(128) % 7 - 3
    a, o = _run("oracle", reduce_src, 2, 64, [("i32", data), ("i32", np.zeros(2))])
    out["kat_general_in"], out["kat_general_a"], out["kat_general_out"] = data.astype(np.int32), a, o
    vall = "__global__ void v(global i32* a, global i32* out) { out[threadIdx.x] = vote_all(a[threadIdx.x] > 0); }"
    _, o = _run("oracle", vall, 1, 32, [("i32", np.ones(32)), ("i32", np.zeros(32))])
    out["kat_vote_all_out"] = o
    vany = "__global__ void v(global i32* a, global i32* out) { out[threadIdx.x] = vote_any(a[threadIdx.x] == 9); }"
    d = np.zeros(64)
    d[37] = 9
    _, o = _run("oracle", vany, 1, 64, [("i32", d), ("i32", np.zeros(64))])
    out["kat_vote_any_in"], out["kat_vote_any_out"] = d.astype(np.int32), o
    shfl = "__global__ void s(global i32* a, global i32* out) { out[threadIdx.x] = shfl_down(a[threadIdx.x], 1); }"
    _, o = _run("oracle", shfl, 1, 32, [("i32", np.arange(32)), ("i32", np.zeros(32))])
    out["kat_shfl_out"] = o
    return out


def c1c2_pin() -> dict:
    out = {}
    n, grid, block = 1 << 14, 8, 256
    for gen in ("i32_full", "i32_small"):
        a = synthetic.generate(gen, n, seed=7)
        _, p1 = _run("oracle", C1_I32, grid, block, [("i32", a), ("i32", np.zeros(grid * 8))], [n])
        _, p2 = _run("launch", C1_I32, grid, block, [("i32", a), ("i32", np.zeros(grid * 8))], [n])
        assert np.array_equal(p1, p2)
        out[f"{gen}_partials"] = p1
    f = synthetic.generate("f32_unit", n, seed=7)
    _, p1 = _run("oracle", C1_F32, grid, block, [("f32", f), ("f32", np.zeros(grid * 8))], [n])
    _, p2 = _run("launch", C1_F32, grid, block, [("f32", f), ("f32", np.zeros(grid * 8))], [n])
    assert np.array_equal(p1.view(np.int32), p2.view(np.int32))
    out["f32_unit_partials"] = p1
    out["meta"] = np.array([n, grid, block, 7], dtype=np.int64)
    return out


def c3_pin() -> dict:
    n, grid, block = 1 << 12, 16, 256
    a = synthetic.generate("i32_full", n, seed=3)
    _, o1 = _run("oracle", C3_WARP_PREFIX, grid, block, [("i32", a), ("i32", np.zeros(n))])
    _, o2 = _run("launch", C3_WARP_PREFIX, grid, block, [("i32", a), ("i32", np.zeros(n))])
    assert np.array_equal(o1, o2)
    return {"warp_prefix_out": o1, "meta": np.array([n, grid, block, 3], dtype=np.int64)}


C4_COMPACT_SERIAL = """
__global__ void compact_gt0(global i32* a, global i32* out, global i32* count, i32 n) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        i32 m = 0;
        for (i32 i = 0; i < n; i = i + 1) {
            if (a[i] > 0) {
                out[m] = a[i];
                m = m + 1;
            }
        }
        count[0] = m;
    }
}
"""

C5_HIST_PER_BIN = """
__global__ void hist256(global i32* a, global i32* bins, i32 n) {
    i32 b = threadIdx.x + blockIdx.x * blockDim.x;
    i32 c = 0;
    for (i32 i = 0; i < n; i = i + 1) {
        if (a[i] == b) {
            c = c + 1;
        }
    }
    bins[b] = c;
}
"""


def c4c5_pin() -> dict:
    out = {}
    cases = [("i32_full", 0, 1 << 12, 5), ("i32_select", 0, 2000, 6), ("i32_select", 10, 2000, 7),
             ("i32_select", 500, 2000, 8), ("i32_select", 1000, 2000, 9)]
    for gen, param, n, seed in cases:
        a = synthetic.generate(gen, n, seed=seed, param=param)
        bufs = [("i32", a), ("i32", np.zeros(n)), ("i32", np.zeros(1))]
        _, o1, c1 = _run("oracle", C4_COMPACT_SERIAL, 1, 32, bufs, [n])
        _, o2, c2 = _run("launch", C4_COMPACT_SERIAL, 1, 32, bufs, [n])
        assert np.array_equal(o1, o2) and np.array_equal(c1, c2)
        tag = f"c4_{gen}_{param}"
        out[f"{tag}_in"], out[f"{tag}_out"], out[f"{tag}_count"] = a, o1[:int(c1[0])], c1
    for gen, param, n, seed in (("u8_uniform", 0, 1 << 12, 5), ("u8_const", 0, 1000, 6),
                                ("u8_geom", 0, 3000, 7)):
        a8 = synthetic.generate(gen, n, seed=seed, param=param)
        a = a8.astype(np.int32)  # the DSL has no u8: bytes widened to i32
        bufs = [("i32", a), ("i32", np.zeros(256))]
        _, b1 = _run("oracle", C5_HIST_PER_BIN, 1, 256, bufs, [n])
        _, b2 = _run("launch", C5_HIST_PER_BIN, 1, 256, bufs, [n])
        assert np.array_equal(b1, b2)
        tag = f"c5_{gen}"
        out[f"{tag}_in"], out[f"{tag}_bins"] = a8, b1
    return out


def random_kernels() -> dict:
    """tests/test_random_diff.py:13-43 restated: seeds 0-149 (grid 1), 150-179
    (specialized: same outputs), 180-199 (grid 3); warp 4, block 8."""
    from warpfold.randgen import generate_kernel
    warp, block = 4, 8
    out = []
    for seed in range(200):
        grid = 3 if seed >= 180 else 1
        src = generate_kernel(seed, warp_size=warp, block_size=block)
        n = grid * block
        gin = (np.arange(n) * 3 - 7).astype(np.int32)
        o1 = _run("oracle", src, grid, block, [("i32", gin), ("i32", np.zeros(n))], [2], warp=warp)
        o2 = _run("launch", src, grid, block, [("i32", gin), ("i32", np.zeros(n))], [2], warp=warp)
        assert all(np.array_equal(a, b) for a, b in zip(o1, o2)), seed
        out.append({"seed": seed, "grid": grid, "block": block, "warp": warp, "scalar": 2,
                    "source": src, "gin": gin.tolist(),
                    "gin_out": o1[0].astype(np.int32).tolist(),
                    "gout": o1[1].astype(np.int32).tolist()})
    return {"source": "warpfold randgen.generate_kernel + run_oracle (cross-checked with "
                      "launch(hybrid_transform(...)))", "kernels": out}


def acceptance_fuzz() -> dict:
    """The reference's acceptance criterion 5 (tests/test_acceptance.py:
    218-236): 1000 fuzzer kernels at warp 4, block 8, gin = 5*i - 9."""
    from warpfold.randgen import generate_kernel
    out = []
    for seed in range(1000):
        src = generate_kernel(seed, warp_size=4, block_size=8)
        gin = (np.arange(8) * 5 - 9).astype(np.int32)
        o = _run("oracle", src, 1, 8, [("i32", gin), ("i32", np.zeros(8))], [2], warp=4)
        out.append([seed, src, o[0].astype(np.int32).tolist(), o[1].astype(np.int32).tolist()])
    return {"source": "warpfold tests/test_acceptance.py criterion 5 inputs; outputs from "
                      "run_oracle", "cases": out}


def corpus_golden() -> tuple[dict, dict]:
    arrays, manifest = {}, {}
    for k in corpus.ALL:
        for grid, block, warp in ((2, 64, 32), (3, 32, 32), (2, 8, 4), (1, 16, 8)):
            mem, args = k.build(grid, block, 0)
            kernel = k.kernel()
            ids = [a for p, a in zip(kernel.params, args) if p.is_buffer]
            kinds = [p.kind for p in kernel.params if p.is_buffer]
            tag = f"{k.name}__g{grid}b{block}w{warp}"
            for i, (bid, kind) in enumerate(zip(ids, kinds)):
                arrays[f"{tag}__in{i}"] = mem.view(bid, kind).copy()
            cfg = LaunchConfig(grid_size=grid, block_size=block, warp_size=warp, workers=1)
            run_oracle(kernel, cfg, bind_args(kernel.params, mem, args))
            for i, (bid, kind) in enumerate(zip(ids, kinds)):
                arrays[f"{tag}__out{i}"] = mem.view(bid, kind).copy()
            manifest[tag] = {"kernel": k.name, "grid": grid, "block": block, "warp": warp,
                             "kinds": kinds,
                             "args": [("buf", kernel.params.index(p)) if p.is_buffer
                                      else ("scalar", a if not isinstance(a, np.floating)
                                            else float(a))
                                      for p, a in zip(kernel.params, args)],
                             "source": k.source}
    return arrays, manifest


def corpus_traces() -> dict:
    """ExecTrace counts from run_oracle (interp/oracle.py:113-136) for every
    corpus configuration, plus each kernel's uid -> IR-class catalogue as
    cfg/build.py allocates it (pins the GPU trace build's uid numbering)."""
    from warpfold import ExecTrace
    from warpfold.cfg.build import build_cfg
    out = {"runs": {}, "kernels": {}}
    extra = [("C1_I32", C1_I32), ("C1_F32", C1_F32), ("C3_WARP_PREFIX", C3_WARP_PREFIX)]
    for name, src in [(k.name, k.source) for k in corpus.ALL] + extra:
        cfg = build_cfg(parse_module(src).kernel())
        kinds = {}
        for b in cfg.blocks.values():
            for i in b.instrs:
                kinds[str(i.uid)] = type(i).__name__
            kinds[str(b.term.uid)] = type(b.term).__name__
        out["kernels"][name] = {"uid_kinds": kinds, "max_uid": cfg._next_uid}
    for k in corpus.ALL:
        for grid, block, warp in ((2, 64, 32), (3, 32, 32), (2, 8, 4), (1, 16, 8)):
            mem, args = k.build(grid, block, 0)
            kernel = k.kernel()
            cfg = LaunchConfig(grid_size=grid, block_size=block, warp_size=warp, workers=1)
            tr = ExecTrace()
            run_oracle(kernel, cfg, bind_args(kernel.params, mem, args), tr)
            run = {"instr": {str(u): c for u, c in sorted(tr.instr_counts.items())},
                   "term": {str(u): c for u, c in sorted(tr.term_counts.items())}}
            if tr.barrier_arrivals:  # interp/oracle.py:207 (warp), :237 (block)
                run["arrivals"] = {str(u): [sorted(s) for s in sets]
                                   for u, sets in sorted(tr.barrier_arrivals.items())}
            out["runs"][f"{k.name}__g{grid}b{block}w{warp}"] = run
    return out


def diff_pipeline_expected() -> str:
    """The reference's own `run --json` output for tests/data/diff_pipeline.json
    (oracle engine): the committed expected dumps of the GPU `diff` command."""
    from warpfold.runtime.hostdesc import run_description
    data = HERE.parent / "data"
    cfg = LaunchConfig(grid_size=1, block_size=32, warp_size=32, workers=1)
    _, dumps = run_description(data / "diff_pipeline.json", cfg, engine="oracle")
    _, dumps2 = run_description(data / "diff_pipeline.json", cfg, engine="mpmd")
    assert dumps == dumps2  # both reference engines agree on this program
    return "".join(json.dumps(d) + "\n" for d in dumps)


def main() -> None:
    if "--diff-only" in sys.argv:
        (HERE.parent / "data" / "diff_pipeline.expected.jsonl").write_text(diff_pipeline_expected())
        return
    if "--random-only" in sys.argv:
        (HERE / "random_kernels.json").write_text(json.dumps(random_kernels()))
        (HERE / "acceptance_fuzz.json").write_text(json.dumps(acceptance_fuzz()))
        return
    if "--c4c5-only" in sys.argv:
        np.savez_compressed(HERE / "c4c5_pin.npz", **c4c5_pin())
        (HERE / "C4_COMPACT_SERIAL.spk").write_text(C4_COMPACT_SERIAL)
        (HERE / "C5_HIST_PER_BIN.spk").write_text(C5_HIST_PER_BIN)
        return
    if "--traces-only" in sys.argv:
        (HERE / "corpus_traces.json").write_text(json.dumps(corpus_traces(), indent=0))
        return
    (HERE / "corpus_traces.json").write_text(json.dumps(corpus_traces(), indent=0))
    (HERE / "warp_semantics.json").write_text(json.dumps(warp_semantics(), indent=1))
    np.savez_compressed(HERE / "oracle_kat.npz", **oracle_kat())
    np.savez_compressed(HERE / "c1c2_pin.npz", **c1c2_pin())
    np.savez_compressed(HERE / "c3_pin.npz", **c3_pin())
    np.savez_compressed(HERE / "c4c5_pin.npz", **c4c5_pin())
    (HERE / "random_kernels.json").write_text(json.dumps(random_kernels()))
    (HERE / "acceptance_fuzz.json").write_text(json.dumps(acceptance_fuzz()))
    arrays, manifest = corpus_golden()
    np.savez_compressed(HERE / "corpus.npz", **arrays)
    (HERE / "corpus_manifest.json").write_text(json.dumps(manifest, indent=1))
    (HERE / "C1_I32.spk").write_text(C1_I32)
    (HERE / "C1_F32.spk").write_text(C1_F32)
    (HERE / "C3_WARP_PREFIX.spk").write_text(C3_WARP_PREFIX)
    (HERE / "C4_COMPACT_SERIAL.spk").write_text(C4_COMPACT_SERIAL)
    (HERE / "C5_HIST_PER_BIN.spk").write_text(C5_HIST_PER_BIN)
    (HERE.parent / "data" / "diff_pipeline.expected.jsonl").write_text(diff_pipeline_expected())
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
