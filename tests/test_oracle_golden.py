"""The oracle against the reference's own golden vectors (CPU only).

Pins oracle/semantics.py, oracle/numpy_oracle.py and oracle/collapse_ref.c
to outputs produced by warpfold itself (tests/golden/make_golden.py) and to
the reference's known-answer tests (tests/test_oracle.py:41-89,
tests/test_warp_lower.py:109-138)."""

import itertools
import json

import numpy as np
import pytest

from oracle import cref, numpy_oracle as no, semantics, synthetic


@pytest.fixture(scope="module")
def sem(golden):
    return json.loads((golden / "warp_semantics.json").read_text())


def test_shuffle_down_table_matches_reference(sem):
    t = sem["shfl_down"]
    buf = t["buffer"]
    for lane in range(32):
        for j, off in enumerate(t["offsets"]):
            assert semantics.shuffle_down(buf, lane, off, 32) == t["table"][lane][j]


def test_reduce_vote_exhaustive_matches_reference(sem):
    for width, rows in sem["reduce_vote"].items():
        for m, want_all, want_any in rows:
            bits = [(m >> k) & 1 for k in range(int(width))]
            assert semantics.reduce_vote(bits, "all") == want_all
            assert semantics.reduce_vote(bits, "any") == want_any


def test_reduce_vote_enumerated():  # reference tests/test_warp_lower.py:113-117
    for width in (4, 8):
        for bits in itertools.product((0, 1), repeat=width):
            assert semantics.reduce_vote(list(bits), "all") == (1 if all(bits) else 0)
            assert semantics.reduce_vote(list(bits), "any") == (1 if any(bits) else 0)


def test_collective_model_reproduces_oracle_kats(golden):
    kat = np.load(golden / "oracle_kat.npz")
    out = semantics.collective("shfl_down", np.arange(32), None, 1, 32, 32, 0xFFFFFFFF)
    assert np.array_equal(out, kat["kat_shfl_out"])
    out = semantics.collective("vote_all", (np.ones(32) > 0).astype(int), None, 0, 32, 32, 0xFFFFFFFF)
    assert np.array_equal(out, kat["kat_vote_all_out"])
    pred = (kat["kat_vote_any_in"] == 9).astype(int)
    out = semantics.collective("vote_any", pred, None, 0, 64, 32, 0xFFFFFFFF)
    assert np.array_equal(out, kat["kat_vote_any_out"])
    # reduce_warp KAT: lane 0 of warp 0 holds the 5-round shfl_down sum
    data = kat["kat_general_in"]
    for b in range(2):
        assert kat["kat_general_out"][b] == data[64 * b:64 * b + 32].sum()
    assert kat["kat_ones_out"][0] == 32


def test_collective_model_resolve_matches_reference_resolver():
    rng = np.random.default_rng(1)
    for _ in range(50):
        vals = rng.integers(-5, 5, 32).tolist()
        offs = rng.integers(-40, 40, 32).tolist()
        want = semantics.resolve("shfl_down", vals, offs, 32)
        got = semantics.collective("shfl_down", vals, offs, 0, 32, 32, 0xFFFFFFFF)
        assert got.tolist() == want


def test_c1_partials_pinned(golden):
    g = np.load(golden / "c1c2_pin.npz")
    n, grid, block, seed = (int(v) for v in g["meta"])
    for gen in ("i32_full", "i32_small"):
        a = synthetic.generate(gen, n, seed=seed)
        assert np.array_equal(no.reference_partials_i32(a, grid, block), g[f"{gen}_partials"])
        total, parts = cref.reduce_i32(a, grid, block)
        assert np.array_equal(parts, g[f"{gen}_partials"])
        assert total == no.reduce_sum_i32(a)


def test_c2_reference_order_pinned_bitwise(golden):
    g = np.load(golden / "c1c2_pin.npz")
    n, grid, block, seed = (int(v) for v in g["meta"])
    f = synthetic.generate("f32_unit", n, seed=seed)
    parts, total = no.reference_order_f32(f, grid, block)
    assert np.array_equal(parts.view(np.int32), g["f32_unit_partials"].view(np.int32))
    ctotal, cparts = cref.reduce_f32(f, grid, block)
    assert np.array_equal(cparts.view(np.int32), g["f32_unit_partials"].view(np.int32))
    assert np.float32(ctotal) == total
    tol = no.f32_tolerance(n, no.abs_sum(f), chain=n // (grid * block))
    assert abs(float(total) - no.reduce_sum_f32_exact(f)) <= tol


def test_c3_warp_prefix_pinned(golden):
    g = np.load(golden / "c3_pin.npz")
    n, grid, block, seed = (int(v) for v in g["meta"])
    a = synthetic.generate("i32_full", n, seed=seed)
    seg = a.reshape(-1, 32)
    want = np.concatenate([no.scan_inclusive_i32(s) for s in seg])
    assert np.array_equal(g["warp_prefix_out"], want)
    # the global scan composes the warp prefixes with exclusive carries
    full = cref.scan_i32(a)
    carries = np.concatenate([[0], np.cumsum(seg.astype(np.int64).sum(1))[:-1]])
    comp = (want.reshape(-1, 32).astype(np.int64) + carries[:, None]) & 0xFFFFFFFF
    assert np.array_equal(full, comp.astype(np.uint32).view(np.int32).reshape(-1))


def test_corpus_suffix_scan_restatement(golden):
    import json as _j
    man = _j.loads((golden / "corpus_manifest.json").read_text())
    arr = np.load(golden / "corpus.npz")
    tag = "shfl_suffix_scan__g2b64w32"
    m = man[tag]
    a = arr[f"{tag}__in0"]
    out = arr[f"{tag}__out1"]
    # only threadIdx < 32 runs the scan (corpus.py:347-364)
    want = a.copy()
    for b in range(m["grid"]):
        seg = slice(b * 64, b * 64 + 32)
        want[seg] = no.warp_suffix_scan_reference(a[seg])
    assert np.array_equal(out, want)


@pytest.mark.parametrize("n", [0, 1, 2, 31, 32, 33, 255, 4096, 4097, 100003])
def test_c_oracle_matches_numpy(n):
    a = synthetic.generate("i32_full", n, seed=n)
    assert np.array_equal(cref.scan_i32(a), no.scan_inclusive_i32(a))
    assert np.array_equal(cref.compact_gt0_i32(a), no.compact_gt0_i32(a))
    u = synthetic.generate("u8_uniform", n, seed=n)
    assert np.array_equal(cref.hist256_u8(u, 7, 64), no.histogram256_u8(u))
    if n:
        t, _ = cref.reduce_i32(a, 3, 64)
        assert t == no.reduce_sum_i32(a)


def test_synthetic_generators_are_index_hashes():
    for gen in synthetic.GENS:
        a = synthetic.generate(gen, 1000, seed=5, param=300)
        b = synthetic.generate(gen, 600, seed=5, base=400, param=300)
        assert np.array_equal(a[400:], b)
    f = synthetic.generate("f32_unit", 100000, seed=1)
    assert f.min() >= -0.5 and f.max() < 0.5
    s = synthetic.generate("i32_select", 100000, seed=2, param=250)
    assert abs((s > 0).mean() - 0.25) < 0.01
    assert (synthetic.generate("i32_select", 1000, param=0) <= 0).all()
    assert (synthetic.generate("i32_select", 1000, param=1000) > 0).all()
    sm = synthetic.generate("i32_small", 100000)
    assert sm.min() == -10 and sm.max() == 10


def test_splitmix64_known_values():
    # splitmix64 reference outputs for state increments from 0 (Vigna)
    h = synthetic.splitmix64(np.array([0], dtype=np.uint64))
    assert int(h[0]) == 0xE220A8397B1DCDAF


def test_f32_tolerance_contract():
    assert no.f32_tolerance(1 << 30, 1.0) == pytest.approx(60 * 2.0 ** -24)
    assert no.f32_tolerance(1, 5.0) == 0.0



def test_c4_compaction_pinned(golden):
    """Ordered compaction: the oracle reproduces the reference's own serial
    in-order compaction kernel (C4_COMPACT_SERIAL.spk via run_oracle and
    launch(hybrid_transform)) at 0/1/50/100 % selectivity."""
    g = np.load(golden / "c4c5_pin.npz")
    cases = [k[:-3] for k in g.files if k.startswith("c4_") and k.endswith("_in")]
    assert len(cases) == 5
    for tag in cases:
        want = g[f"{tag}_out"]
        assert int(g[f"{tag}_count"][0]) == len(want)
        assert np.array_equal(no.compact_gt0_i32(g[f"{tag}_in"]), want), tag


def test_c5_histogram_pinned(golden):
    """256-bin byte histogram: the oracle reproduces the reference's
    one-thread-per-bin counting kernel (C5_HIST_PER_BIN.spk) on uniform,
    constant and geometric bytes."""
    g = np.load(golden / "c4c5_pin.npz")
    cases = [k[:-3] for k in g.files if k.startswith("c5_") and k.endswith("_in")]
    assert len(cases) == 3
    for tag in cases:
        got = no.histogram256_u8(g[f"{tag}_in"])
        assert np.array_equal(got.astype(np.int64), g[f"{tag}_bins"].astype(np.int64)), tag
