"""Host-side logic that needs no GPU: the launch contract (config
validation, argument binding, error mapping) and the C ABI's exports.

Mirrors the reference's runtime tests (tests/test_runtime.py:65-78 arity /
kind errors) and config rules (config.py:26-41)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2112_10034_b200 import LaunchConfig, errors
from paper_2112_10034_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "warpfold_b200.h"


def header_functions() -> set:
    text = HEADER.read_text()
    return set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(wf_\w+)\s*\(", text, re.M))


# ---- config (reference config.py:26-41 + B200 extensions) ------------------

@pytest.mark.parametrize("kw,msg", [
    (dict(grid_size=-1), "grid size must be >= 0"),
    (dict(block_size=0), "block size must be >= 1"),
    (dict(warp_size=0), "warp size must be >= 1"),
    (dict(workers=0), "workers must be >= 1"),
    (dict(mode="x"), "mode must be one of"),
    (dict(block_size=2048), "block size must be <= 1024"),
    (dict(warp_size=3), "warp size must be one of"),
    (dict(shared_bytes=300 * 1024), "shared_bytes must be in"),
])
def test_config_rejects(kw, msg):
    with pytest.raises(errors.ConfigError, match=msg):
        LaunchConfig(**kw).validate()


def test_config_partial_warps_extension():
    cfg = LaunchConfig(block_size=48)
    cfg.validate(hierarchical=True)  # B200 path accepts partial warps
    strict = LaunchConfig(block_size=48, allow_partial_warps=False)
    with pytest.raises(errors.ConfigError, match="divisible by warp size"):
        strict.validate(hierarchical=True)
    assert LaunchConfig(block_size=256).warps_per_block == 8


def test_error_hierarchy_matches_reference():
    assert issubclass(errors.BarrierViolation, errors.ExecutionError)
    assert issubclass(errors.SemanticError, errors.ParseError)
    for name in ("ConfigError", "LaunchError", "ExecutionError", "UnsupportedFeatureError",
                 "TransformError", "DivergenceError"):
        assert issubclass(getattr(errors, name), errors.WarpfoldError)
    e = errors.ParseError("bad", 3, 4)
    assert str(e) == "3:4: bad" and e.line == 3


# ---- bind_args (reference runtime/launch.py:28-46) -------------------------

class _FakeMem:
    def bind_view(self, buffer_id, kind):
        return np.zeros(4, dtype=np.int32)


def test_bind_args_messages():
    from paper_2112_10034_b200.runtime import Param, bind_args
    params = [Param("a", "i32", True), Param("n", "i32", False), Param("s", "f32", False)]
    with pytest.raises(errors.LaunchError, match="kernel takes 3 arguments, got 2"):
        bind_args(params, _FakeMem(), [1, 2])
    with pytest.raises(errors.LaunchError, match="'a' must be a buffer id"):
        bind_args(params, _FakeMem(), [1.5, 2, 1.0])
    with pytest.raises(errors.LaunchError, match="'n' must be an i32 scalar"):
        bind_args(params, _FakeMem(), [1, True, 1.0])
    with pytest.raises(errors.LaunchError, match="'s' must be an f32 scalar"):
        bind_args(params, _FakeMem(), [1, 2, "x"])
    b = bind_args(params, _FakeMem(), [1, 2, 0.5])
    assert b["n"] == 2 and b["s"] == np.float32(0.5)


def test_program_registry_signatures():
    from paper_2112_10034_b200.runtime import PROGRAMS, warp_program
    assert set(PROGRAMS) == {"reduce_sum_i32", "reduce_sum_f32", "scan_inclusive_i32",
                             "compact_gt0_i32", "histogram256_u8"}
    assert [p.name for p in PROGRAMS["compact_gt0_i32"].params] == ["a", "out", "count", "n"]
    assert [p.name for p in warp_program("shfl_down").params] == ["a", "b", "out"]
    assert [p.name for p in warp_program("vote_any", per_lane_operand=False).params] == ["a", "out"]


# ---- the C ABI -------------------------------------------------------------

@pytest.fixture(scope="module")
def lib():
    from paper_2112_10034_b200 import build
    build.build_library()
    return _lib.load()


def test_library_exports_every_header_symbol(lib):
    declared = header_functions()
    assert len(declared) >= 20
    raw = ctypes.CDLL(str(_lib.lib_path()))
    for name in sorted(declared):
        assert hasattr(raw, name), f"{name} declared in the header but not exported"
    assert declared == set(_lib.SIGNATURES), "ctypes table and header disagree"


def test_abi_metadata(lib):
    assert lib.wf_abi_version() == 1
    assert b"sm_100a" in lib.wf_version()
    assert lib.wf_workspace_bytes(_lib.OP_REDUCE_SUM_F32, 1 << 30, 256) >= 256
    # scan workspace: 8 KiB header (two-pass chunk counters) + one descriptor per 4096-element tile, each on
    # its own 128-byte line (look-back polling must not share lines)
    assert lib.wf_workspace_bytes(_lib.OP_SCAN_INCLUSIVE_I32, 1 << 28, 256) == 8192 + (1 << 16) * 128
    assert lib.wf_workspace_bytes(_lib.OP_HISTOGRAM256_U8, 1, 256) == 256 + 2048


def test_abi_argument_errors_map_to_reference_exceptions(lib):
    # all of these are rejected before any CUDA call, so they run without a GPU
    rc = lib.wf_reduce_sum_i32(None, 0, 16, 100, 0, None, 0, None)
    assert rc == _lib.WF_ERR_CONFIG and "block size" in _lib.last_error()
    with pytest.raises(errors.ConfigError):
        _lib.check(rc)
    rc = lib.wf_reduce_sum_f32(None, 10, 16, 256, 0, None, 0, None)
    assert rc == _lib.WF_ERR_ARG
    with pytest.raises(errors.LaunchError, match="input pointer"):
        _lib.check(rc)
    rc = lib.wf_reduce_sum_f32(64, 10, 16, 256, 0, None, 0, None)
    assert rc == _lib.WF_ERR_WORKSPACE
    rc = lib.wf_warp_collective(99, None, None, 0, None, 32, 32, 32, 0xFFFFFFFF, None)
    with pytest.raises(errors.UnsupportedFeatureError):
        _lib.check(rc)
    rc = lib.wf_warp_collective(0, None, None, 0, None, 33, 32, 32, 0xFFFFFFFF, None)
    assert rc == _lib.WF_ERR_CONFIG and "multiple of the block size" in _lib.last_error()
    rc = lib.wf_warp_collective(0, None, None, 0, None, 32, 32, 3, 0xFFFFFFFF, None)
    assert rc == _lib.WF_ERR_CONFIG
    rc = lib.wf_compact_gt0_i32(64, 1 << 33, 64, 64, None, 0, None)
    assert rc == _lib.WF_ERR_ARG and "2^32" in _lib.last_error()
    rc = lib.wf_fill_synthetic(42, None, 0, 0, 0, 0, None)
    assert rc == _lib.WF_ERR_UNSUPPORTED


def test_fused_exchange_entry_points_validate_before_launch(lib):
    """The *_mg entry points reject bad mailbox arguments before any CUDA
    call (fake, aligned device addresses; no GPU needed)."""
    ws, wsb, ptr = 256, 1 << 20, 64
    # (in, n, out2, block, grid, ws, ws_bytes, peers, mailbox, cap, rank, world, epoch, err, stream)
    rc = lib.wf_reduce_sum_i32_exscan_mg(ptr, 10, ptr, 256, 0, ws, wsb, None, ptr, 1, 0, 1, 1, ptr, None)
    assert rc == _lib.WF_ERR_ARG and "NULL" in _lib.last_error()
    rc = lib.wf_reduce_sum_i32_exscan_mg(ptr, 10, ptr, 256, 0, ws, wsb, ptr, ptr, 0, 0, 1, 1, ptr, None)
    assert rc == _lib.WF_ERR_ARG and "cap 0 < 1" in _lib.last_error()
    rc = lib.wf_reduce_sum_i32_exscan_mg(ptr, 10, ptr, 256, 0, ws, wsb, ptr, ptr, 1, 0, 1, 0, ptr, None)
    assert rc == _lib.WF_ERR_ARG and "epoch" in _lib.last_error()
    rc = lib.wf_reduce_sum_i32_exscan_mg(ptr, 10, ptr, 256, 0, ws, wsb, ptr, ptr, 1, 3, 2, 1, ptr, None)
    assert rc == _lib.WF_ERR_ARG and "out of range" in _lib.last_error()
    rc = lib.wf_reduce_sum_i32_exscan_mg(ptr, 10, ptr, 100, 0, ws, wsb, ptr, ptr, 1, 0, 1, 1, ptr, None)
    assert rc == _lib.WF_ERR_CONFIG
    # (in, n, bins, ws, ws_bytes, peers, mailbox, cap, rank, world, epoch, err, stream)
    rc = lib.wf_histogram256_u8_mg(ptr, 10, ptr, ws, wsb, ptr, ptr, 255, 0, 1, 1, ptr, None)
    assert rc == _lib.WF_ERR_ARG and "cap 255 < 256" in _lib.last_error()
    # (in, n, out, counts3, ws, ws_bytes, peers, mailbox, cap, rank, world, epoch, err, stream)
    rc = lib.wf_compact_gt0_i32_mg(ptr, 1 << 33, ptr, ptr, ws, 1 << 40, ptr, ptr, 1, 0, 1, 1, ptr,
                                   None)
    assert rc == _lib.WF_ERR_ARG and "2^32" in _lib.last_error()
    rc = lib.wf_compact_gt0_i32_mg(ptr, 10, ptr, None, ws, wsb, ptr, ptr, 1, 0, 1, 1, ptr, None)
    assert rc == _lib.WF_ERR_ARG and "counts" in _lib.last_error()


def test_cuda_error_codes_map_to_execution_error():
    with pytest.raises(errors.ExecutionError, match="CUDA error 700"):
        _lib.check(700, "illegal address")


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setenv("WF_LIB", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(errors.NativeLibraryMissing, match="no CPU fallback"):
        _lib.load()


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2112_10034_b200"
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle\b", text, re.M), py


# ---- diff report logic (reference interp/diff.py:48-72) --------------------

def test_compare_memory_and_dumps():
    from paper_2112_10034_b200.diff import compare_dumps, compare_memory
    a = np.arange(8, dtype=np.int32)
    f = np.linspace(0, 1, 8).astype(np.float32)
    ref = {1: a.tobytes(), 2: f.tobytes()}
    assert compare_memory(ref, dict(ref), {1: "i32", 2: "f32"}).equal
    b = a.copy()
    b[3] = 99
    rep = compare_memory(ref, {1: b.tobytes(), 2: f.tobytes()}, {1: "i32", 2: "f32"})
    assert not rep.equal and rep.divergence == {"buffer": 1, "element": 3, "reference": 3,
                                                "transformed": 99}
    assert rep.detail == "buffer 1 diverges at element 3: reference=3 transformed=99"
    g = f.copy()
    g[2] += 1e-5
    got = {1: a.tobytes(), 2: g.tobytes()}
    assert not compare_memory(ref, got, {1: "i32", 2: "f32"}).equal
    assert compare_memory(ref, got, {1: "i32", 2: "f32"}, fp_tol=1e-4).equal
    rep = compare_memory(ref, {1: a.tobytes()[:-1], 2: f.tobytes()}, {})
    assert rep.divergence["detail"] == "length mismatch"
    e = [{"buffer": "x", "kind": "i32", "values": [1, 2, 3]}]
    assert compare_dumps(e, [{"buffer": "x", "kind": "i32", "values": [1, 2, 3]}]).equal
    rep = compare_dumps(e, [{"buffer": "x", "kind": "i32", "values": [1, 5, 3]}])
    assert rep.divergence["element"] == 1
    assert not compare_dumps(e, []).equal


def test_refcheck_is_checker_only():
    """The reference is reached only by the diff command's checker module;
    no op / runtime / kernel module imports it."""
    pkg = ROOT / "paper_2112_10034_b200"
    uses = re.compile(r"^\s*(from\s+\.+\s+import\s+.*\brefcheck\b|from\s+\.refcheck\b|"
                      r"import\s+.*refcheck)", re.M)
    assert [p.name for p in pkg.rglob("*.py") if uses.search(p.read_text())] == ["__main__.py"]
    imports = re.compile(r"^\s*(from\s+warpfold[\s.]|import\s+warpfold\b)", re.M)
    assert [p.name for p in pkg.rglob("*.py")
            if imports.search(p.read_text()) and p.name != "refcheck.py"] == []


def build_c_consumer(tmp_path):
    """tests/c_consumer/abi_consumer.c as a plain C99 program linked against
    the library and the CUDA runtime (-Wall -Wextra -Werror: the header is
    valid C)."""
    import subprocess
    exe = tmp_path / "abi_consumer"
    lib_dir = _lib.lib_path().parent
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-O2", f"-I{ROOT / 'include'}",
           str(ROOT / "tests" / "c_consumer" / "abi_consumer.c"), f"-L{lib_dir}",
           f"-l:{_lib.lib_path().name}", f"-Wl,-rpath,{lib_dir}", "-L/usr/local/cuda/lib64",
           "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_consumer_links_and_maps_errors(tmp_path):
    """The boundary from C: no Python, no torch in the process."""
    import subprocess
    r = subprocess.run([str(build_c_consumer(tmp_path)), "cpu"], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "OK cpu", r.stderr
