"""DSL front end on CPU: parsing (reference tests/test_parser.py shapes),
kind checking, mode resolution, and that the generated CUDA compiles for
sm_100a for every corpus kernel."""

import json
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import pytest

from paper_2112_10034_b200 import LaunchConfig, errors
from paper_2112_10034_b200.dsl import hybrid_transform, nodes as n, parse_module

GOLDEN = Path(__file__).resolve().parent / "golden"
CORPUS = json.loads((GOLDEN / "corpus_manifest.json").read_text())
SOURCES = {m["kernel"]: m["source"] for m in CORPUS.values()}

CODE1 = """
__global__ void reduce(global i32* a, global i32* out) {
    i32 tid = threadIdx.x + blockIdx.x * blockDim.x;
    i32 val = a[tid];
    for (i32 offset = 16; offset > 0; offset = offset / 2) {
        val = val + shfl_down(0xffffffff, val, offset);
    }
    if (threadIdx.x % 32 == 0) { out[tid / 32] = val; }
}
"""


def test_parse_paper_code1_and_corpus():
    k = parse_module(CODE1).kernel()
    assert k.name == "reduce" and [p.name for p in k.params] == ["a", "out"]
    assert n.uses_warp_features(k)
    for name, src in SOURCES.items():
        kk = parse_module(src).kernel()
        assert kk.name == name


def test_full_mask_literals_normalise():
    a = parse_module(CODE1).kernel()
    b = parse_module(CODE1.replace("0xffffffff, ", "")).kernel()
    c = parse_module(CODE1.replace("0xffffffff", "-1")).kernel()
    assert a == b == c  # structural equality (reference dsl/nodes.py:1-5)


def test_extensions_parse():
    src = """
    __global__ void k(global i32* a, global i32* out, i32 m) {
        extern shared i32 buf[];
        i32 t = threadIdx.x;
        buf[t] = a[t];
        __syncwarp(m);
        out[t] = __shfl_up_sync(m, a[t], 1) + shfl_xor(a[t], 3) + __ballot_sync(m, a[t] > 0)
                 + shfl_idx(a[t], 0) + reduce_add(a[t]) + __any_sync(-1, a[t]);
    }"""
    k = parse_module(src).kernel()
    calls = [e for s in n.walk_stmts(k.body) if isinstance(s, n.Assign)
             for e in n.walk_exprs(s.expr) if isinstance(e, n.CollectiveCall)]
    assert [c.op for c in calls] == ["shfl_up", "shfl_xor", "ballot", "shfl_idx", "reduce_add",
                                     "vote_any"]
    assert calls[0].mask == n.VarRef("m") and calls[-1].mask is None


@pytest.mark.parametrize("src,exc,msg", [
    ("__global__ void k(global i32* a) { grid_sync(); }", errors.UnsupportedFeatureError, "grid"),
    ("__global__ void k(global i32* a) { a[0] = a[1] << 2; }", errors.UnsupportedFeatureError, "shift"),
    ("__global__ void k(global u8* a) { }", errors.UnsupportedFeatureError, "u8"),
    ("__global__ void k(global i32* a) { a[0] = 1 }", errors.ParseError, "expected ';'"),
    ("__global__ void k(global i32* a) { b[0] = 1; }", errors.SemanticError, "unknown identifier 'b'"),
    ("__global__ void k(global i32* a) { i32 x; i32 x; }", errors.SemanticError, "redeclaration"),
    ("__global__ void k(global i32* a, global f32* f) { a[0] = f[0]; }", errors.SemanticError,
     "cannot assign f32 value to i32"),
    ("__global__ void k(global f32* f) { f[0] = f[1] % 2.0; }", errors.SemanticError, "'%'"),
    ("__global__ void k(global i32* a, i32 n) { n = 1; }", errors.SemanticError,
     "cannot assign to parameter"),
    ("__global__ void k(global i32* a) { if (1.0) { a[0] = 1; } }", errors.SemanticError,
     "if condition must be i32"),
    ("__global__ void k(global i32* a) { a[0] = foo(1); }", errors.ParseError, "unknown function"),
])
def test_rejections(src, exc, msg):
    with pytest.raises(exc, match=msg):
        parse_module(src)


def test_parse_error_positions():
    with pytest.raises(errors.ParseError) as ei:
        parse_module("__global__ void k(global i32* a) {\n  a[0] = = 1;\n}")
    assert ei.value.line == 2


def test_mode_resolution_matches_reference():
    k = parse_module(CODE1).kernel()
    cfg = LaunchConfig(grid_size=1, block_size=32)
    assert hybrid_transform(k, cfg).mode == "hier"
    with pytest.raises(errors.UnsupportedFeatureError, match="flat translation"):
        hybrid_transform(k, cfg, mode="flat")
    flat = parse_module(SOURCES["veccopy"]).kernel()
    assert hybrid_transform(flat, cfg).mode == "flat"


def test_codegen_semantics_markers():
    k = parse_module("""
    __global__ void k(global i32* a, global f32* f, i32 n) {
        i32 x;
        f32 y = 1;
        a[0] = a[1] / n + a[2] % n;
        f[0] = f[1] * 0.1 + y;
        a[3] = (a[4] > 0) && (a[5] < 0);
    }""").kernel()
    src = hybrid_transform(k, LaunchConfig(grid_size=1, block_size=32)).source
    assert "wf_div(" in src and "wf_rem(" in src          # trunc div/rem with fault
    assert "__fmul_rn(" in src and "__fadd_rn(" in src     # no FMA contraction
    assert "__int_as_float(0x3dcccccd)" in src             # 0.1f exactly
    assert "wf_land(" in src                               # eager &&
    assert "int v_x = (int)0;" in src                      # zeroed locals
    assert "v_y = wf_f(((int)0x00000001u));" in src        # widening on assignment


def _nvcc(item):
    name, src, tmp = item
    path = tmp / f"{name}.cu"
    path.write_text(src)
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false",
                        "-std=c++17", "-c", "-o", str(tmp / f"{name}.o"), str(path)],
                       capture_output=True, text=True)
    return name, r.returncode, r.stderr


def test_generated_cuda_compiles_for_sm100a(tmp_path):
    items = []
    for tag, m in CORPUS.items():
        k = parse_module(m["source"]).kernel()
        for spec in (False, True):
            cfg = LaunchConfig(grid_size=m["grid"], block_size=m["block"], warp_size=m["warp"],
                               specialize=spec)
            items.append((f"{tag}_{int(spec)}", hybrid_transform(k, cfg).source, tmp_path))
    items = items[::3]  # a representative third keeps the CPU suite fast
    with ThreadPoolExecutor(8) as ex:
        for name, rc, err in ex.map(_nvcc, items):
            assert rc == 0, f"{name}: {err[:2000]}"


def test_cli_transform_emits_cuda(tmp_path):
    from paper_2112_10034_b200.__main__ import main
    out = tmp_path / "k.cu"
    rc = main(["transform", str(GOLDEN / "C1_I32.spk"), "--block-size", "256", "-o", str(out)])
    assert rc == 0 and "wf_shfl_down<int>" in out.read_text()
    bad = tmp_path / "bad.spk"
    bad.write_text("__global__ void k(global i32* a) { a[0] = 1 }")
    assert main(["transform", str(bad)]) == 3  # parse error -> EXIT_TRANSFORM


def test_reference_fuzzer_kernels_parse_check_and_generate():
    """Every kernel of the reference's fuzzer (tests/golden/random_kernels.json)
    goes through this front end: parse, check, CUDA codegen at warp size 4."""
    import json
    from pathlib import Path
    from paper_2112_10034_b200.dsl import codegen, parse_module
    from paper_2112_10034_b200.dsl.checker import check_kernel
    cases = json.loads((Path(__file__).resolve().parent / "golden" / "random_kernels.json")
                       .read_text())["kernels"]
    assert len(cases) == 200
    for c in cases:
        kernel = parse_module(c["source"]).kernel()
        table = check_kernel(kernel)
        src, _ = codegen.generate(kernel, table, warp_size=c["warp"])
        assert "__global__" in src
