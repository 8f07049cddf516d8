"""The reference's own DSL formulations of the hot path, through the drop-in
``launch(hybrid_transform(kernel, cfg), cfg, memory, args)`` (reference
runtime/launch.py:90, passes/pipeline.py:103-179), dispatched by the
structural registry (dsl/patterns.py) to native kernels (csrc/wf_patterns.cu).

Checked against: the reference's own outputs (tests/golden/c1c2_pin.npz,
c3_pin.npz, produced by make_golden.py running warpfold), and the generic
compiled form of the same DSL kernel (the registry switched off), bit for bit
— fp32 partials included — over ragged sizes, grids and the BASELINE sizes."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import numpy_oracle as no, synthetic  # noqa: E402

GOLDEN = Path(__file__).resolve().parent / "golden"
SRC = {k: (GOLDEN / f"{k}.spk").read_text() for k in ("C1_I32", "C1_F32", "C3_WARP_PREFIX")}


@pytest.fixture(scope="module")
def wf():
    from paper_2112_10034_b200 import build
    build.build_library()
    import paper_2112_10034_b200 as wf
    return wf


@pytest.fixture
def calls(monkeypatch):
    """Counts native-pattern dispatches (the registry hit) per launch."""
    from paper_2112_10034_b200.dsl import patterns
    seen = []
    orig = patterns.NativePattern.run

    def spy(self, *a, **k):
        seen.append(self.name)
        return orig(self, *a, **k)

    monkeypatch.setattr(patterns.NativePattern, "run", spy)
    return seen


def _program(src, cfg, generic=False):
    from paper_2112_10034_b200.dsl import hybrid_transform, parse_module
    prog = hybrid_transform(parse_module(src).kernel(), cfg)
    if generic:
        prog.native = None
    return prog


def _partials(wf, src, kind, n, grid, block, fill, generic=False, a_len=None, out_len=None):
    mem = wf.DeviceMemory()
    a = mem.alloc(4 * (a_len if a_len is not None else max(n, 1)))
    out = mem.alloc(4 * (out_len if out_len is not None else max(grid * block // 32, 1)))
    av = mem.device_view(a, kind)
    fill(av)
    cfg = wf.LaunchConfig(grid_size=grid, block_size=block, warp_size=32)
    wf.launch(_program(src, cfg, generic), cfg, mem, [a, out, n])
    return mem.device_view(out, kind)[:grid * block // 32].clone()


def _synth(wf, gen, seed):
    return lambda t: wf.ops.fill_synthetic(gen, t.numel(), seed=seed, out=t)


def test_registry_hits_reference_pins(wf, calls):
    g = np.load(GOLDEN / "c1c2_pin.npz")
    n, grid, block, seed = (int(v) for v in g["meta"])
    for gen, src, kind in (("i32_full", "C1_I32", "i32"), ("i32_small", "C1_I32", "i32"),
                           ("f32_unit", "C1_F32", "f32")):
        got = _partials(wf, SRC[src], kind, n, grid, block, _synth(wf, gen, seed)).cpu().numpy()
        want = g[f"{gen}_partials"]
        assert got.dtype == want.dtype and np.array_equal(got.view(np.int32), want.view(np.int32))
    assert calls == ["warp_partials_sum_i32", "warp_partials_sum_i32", "warp_partials_sum_f32"]


def test_warp_prefix_reference_pin(wf, calls):
    g = np.load(GOLDEN / "c3_pin.npz")
    n, grid, block, seed = (int(v) for v in g["meta"])
    mem = wf.DeviceMemory()
    a, out = mem.alloc(4 * n), mem.alloc(4 * n)
    mem.write(a, synthetic.generate("i32_full", n, seed=seed), "i32")
    cfg = wf.LaunchConfig(grid_size=grid, block_size=block, warp_size=32)
    wf.launch(_program(SRC["C3_WARP_PREFIX"], cfg), cfg, mem, [a, out])
    assert np.array_equal(mem.view(out, "i32"), g["warp_prefix_out"])
    assert calls == ["warp_prefix32_i32"]


CASES = [  # (n, grid, block): ragged n, n < threads, n = 0, negative n, big blocks
    (1, 1, 32), (31, 1, 64), (1000, 3, 96), (4097, 7, 256), ((1 << 20) + 3, 64, 256),
    ((1 << 20), 4096, 256), (123457, 148, 1024), (0, 5, 128), (-7, 2, 64), (5000, 1, 32),
    # one element per DSL thread (the vectorised native path): ragged last
    # segment, whole warps past n, n a multiple of 4 but not of 32
    (100, 2, 64), ((1 << 20) - 5, 4096, 256), (4100, 33, 128), (999, 40, 32),
]


def test_partials_one_element_per_thread_special_values(wf, calls):
    """The vectorised one-element-per-thread path replays the DSL's fp32
    adds exactly: -0.0 (0 + -0.0 = +0.0), infinities and NaN included."""
    vals = torch.tensor([-0.0, 1.5, float("inf"), -2.25, float("-inf"), 3.0e38, 3.0e38, -1e-45,
                         float("nan"), 0.1, -0.0, 7.0], dtype=torch.float32)

    def fill(t):
        t.copy_(vals.repeat(t.numel() // vals.numel() + 1)[:t.numel()].to(t.device))
    for n, grid, block in ((12, 1, 32), (1000, 40, 32), (4096 + 7, 20, 256)):
        got = _partials(wf, SRC["C1_F32"], "f32", n, grid, block, fill)
        want = _partials(wf, SRC["C1_F32"], "f32", n, grid, block, fill, generic=True)
        assert torch.equal(got.view(torch.int32), want.view(torch.int32)), n


@pytest.mark.parametrize("n,grid,block", CASES)
@pytest.mark.parametrize("src,kind,gen", [("C1_I32", "i32", "i32_full"),
                                          ("C1_F32", "f32", "f32_unit")])
def test_partials_native_equals_generic(wf, calls, n, grid, block, src, kind, gen):
    fill = _synth(wf, gen, n & 0xFFFF)
    got = _partials(wf, SRC[src], kind, n, grid, block, fill)
    want = _partials(wf, SRC[src], kind, n, grid, block, fill, generic=True)
    assert calls == [f"warp_partials_sum_{kind}"]
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))


@pytest.mark.parametrize("grid,block", [(1, 32), (3, 96), (148, 256), (4096, 256), (5, 1024),
                                        # larger grids: multi-wave, odd grids, big blocks
                                        (4096, 256 + 32), (4096 + 37, 256), (33000, 32),
                                        (1200, 1024)])
def test_warp_prefix_native_equals_generic(wf, calls, grid, block):
    n = grid * block
    res = []
    for generic in (False, True):
        mem = wf.DeviceMemory()
        a, out = mem.alloc(4 * n), mem.alloc(4 * n)
        wf.ops.fill_synthetic("i32_full", n, seed=grid, out=mem.device_view(a, "i32"))
        cfg = wf.LaunchConfig(grid_size=grid, block_size=block, warp_size=32)
        wf.launch(_program(SRC["C3_WARP_PREFIX"], cfg, generic), cfg, mem, [a, out])
        res.append(mem.device_view(out, "i32").clone())
    assert calls == ["warp_prefix32_i32"]
    assert torch.equal(res[0], res[1])


def test_warp_prefix_misaligned_views(wf):
    """The scalar kernel (4-byte-aligned buffers) against numpy."""
    from paper_2112_10034_b200.dsl import patterns
    pat = patterns.NativePattern("warp_prefix32_i32", "wf_warp_prefix32_i32", "a", "out")
    n = 96 * 37
    x = synthetic.generate("i32_full", n + 1, seed=3)
    a = torch.from_numpy(x).cuda()[1:]
    out = torch.zeros(n + 3, dtype=torch.int32, device="cuda")[3:]
    cfg = type("C", (), {"grid_size": 37, "block_size": 96, "warp_size": 32})()
    pat.run(cfg, {"a": a, "out": out}, torch.cuda.current_stream().cuda_stream)
    seg = x[1:].reshape(-1, 32).astype(np.int64).cumsum(axis=1) & 0xFFFFFFFF
    assert np.array_equal(out.cpu().numpy(), seg.astype(np.uint32).view(np.int32).reshape(-1))


def test_fallbacks_keep_dsl_semantics(wf, calls):
    """Out of the native kernel's preconditions the generic compiled kernel
    runs: other warp size, an out buffer too short (the DSL's fault),
    aliased buffers."""
    from paper_2112_10034_b200.errors import ExecutionError
    fill = _synth(wf, "i32_full", 1)
    # out too short: grid*block/32 = 8 partials, 7 slots -> out-of-bounds write fault
    with pytest.raises(ExecutionError, match="out-of-bounds write"):
        _partials(wf, SRC["C1_I32"], "i32", 4096, 2, 128, fill, out_len=7)
    # a too short: the read fault
    with pytest.raises(ExecutionError, match="out-of-bounds read"):
        _partials(wf, SRC["C1_I32"], "i32", 4096, 2, 128, fill, a_len=4000)
    assert calls == []
    # warp size 8 at hier: generic path, still runs
    mem = wf.DeviceMemory()
    a, out = mem.alloc(4 * 256), mem.alloc(4 * 64)
    mem.write(a, np.ones(256, dtype=np.int32), "i32")
    cfg = wf.LaunchConfig(grid_size=1, block_size=64, warp_size=8)
    wf.launch(_program(SRC["C1_I32"], cfg), cfg, mem, [a, out, 256])
    assert calls == []
    # aliasing: a and out the same buffer
    mem = wf.DeviceMemory()
    a = mem.alloc(4 * 1024)
    mem.write(a, np.ones(1024, dtype=np.int32), "i32")
    cfg = wf.LaunchConfig(grid_size=1, block_size=64, warp_size=32)
    wf.launch(_program(SRC["C1_I32"], cfg), cfg, mem, [a, a, 64])
    assert calls == []


@pytest.mark.slow
def test_reference_formulation_c2_full_size(wf, calls):
    """C2 at 2^30 through the reference's own kernel text: native partials
    bit-identical to the generic compiled kernel, and their fold within the
    SURVEY §8c fp32 bound of the fp64 sum."""
    n, grid, block = 1 << 30, 148 * 8, 256
    fill = _synth(wf, "f32_unit", 1)
    got = _partials(wf, SRC["C1_F32"], "f32", n, grid, block, fill)
    want = _partials(wf, SRC["C1_F32"], "f32", n, grid, block, fill, generic=True)
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    fill(x)
    exact = float(torch.sum(x, dtype=torch.float64))
    absx = float(torch.sum(x.abs(), dtype=torch.float64))
    total = np.float32(0)
    for p in got.cpu().numpy():  # the reference's host fold
        total = np.float32(total + p)
    assert abs(float(total) - exact) <= no.f32_tolerance(n, absx)
    assert calls == ["warp_partials_sum_f32"]


@pytest.mark.slow
def test_reference_formulation_c1_c3_full_size(wf, calls):
    """C1 (2^20, block 256, one element per thread and grid 64) and the warp
    prefix at 2^28: native == generic, bit for bit."""
    fill = _synth(wf, "i32_full", 0)
    for grid in (4096, 64):
        got = _partials(wf, SRC["C1_I32"], "i32", 1 << 20, grid, 256, fill)
        want = _partials(wf, SRC["C1_I32"], "i32", 1 << 20, grid, 256, fill, generic=True)
        assert torch.equal(got, want)
        assert int(got.to(torch.int64).sum()) & 0xFFFFFFFF == no.reduce_sum_i32(
            synthetic.generate("i32_full", 1 << 20, seed=0)) & 0xFFFFFFFF
    n = 1 << 28
    grid, block = n // 256, 256
    res = []
    for generic in (False, True):
        mem = wf.DeviceMemory()
        a, out = mem.alloc(4 * n), mem.alloc(4 * n)
        wf.ops.fill_synthetic("i32_full", n, seed=2, out=mem.device_view(a, "i32"))
        cfg = wf.LaunchConfig(grid_size=grid, block_size=block, warp_size=32)
        wf.launch(_program(SRC["C3_WARP_PREFIX"], cfg, generic), cfg, mem, [a, out])
        res.append(mem.device_view(out, "i32").clone())
        del mem
    assert torch.equal(res[0], res[1])
    assert calls == ["warp_partials_sum_i32"] * 2 + ["warp_prefix32_i32"]
