"""CPU: the structural registry (dsl/patterns.py) recognises the reference's
own formulations of the hot path up to renaming, and nothing else."""

from pathlib import Path

import pytest

from paper_2112_10034_b200.dsl import parse_module, patterns

GOLDEN = Path(__file__).resolve().parent / "golden"


def _k(src):
    return parse_module(src).kernel()


@pytest.mark.parametrize("f,name", [("C1_I32", "warp_partials_sum_i32"),
                                    ("C1_F32", "warp_partials_sum_f32"),
                                    ("C3_WARP_PREFIX", "warp_prefix32_i32")])
def test_reference_kernels_match(f, name):
    m = patterns.match(_k((GOLDEN / f"{f}.spk").read_text()))
    assert m is not None and m.name == name and (m.a, m.out) == ("a", "out")


def test_golden_texts_are_the_templates():
    """The committed reference kernel texts and the registry templates are
    the same kernels (make_golden.py wrote the .spk files)."""
    assert _k((GOLDEN / "C1_I32.spk").read_text()) == _k(patterns.C1_I32)
    assert _k((GOLDEN / "C1_F32.spk").read_text()) == _k(patterns.C1_F32)
    assert _k((GOLDEN / "C3_WARP_PREFIX.spk").read_text()) == _k(patterns.C3_WARP_PREFIX)


def test_renaming_matches_and_roles_follow():
    src = patterns.C1_F32.replace("wsum", "my_reduce").replace("sum", "acc") \
        .replace("global f32* a", "global f32* xs").replace("a[i]", "xs[i]") \
        .replace(" i32 n)", " i32 count)").replace("i < n", "i < count")
    m = patterns.match(_k(src))
    assert m is not None and (m.a, m.out, m.n) == ("xs", "out", "count")


@pytest.mark.parametrize("edit", [
    ("off = 16", "off = 8"),              # different tree
    ("tx % 32 == 0", "tx % 32 == 1"),     # another lane writes
    ("sum = sum + a[i]", "sum = a[i] + sum"),  # other association order (f32)
    ("i32 tx = threadIdx.x;", "i32 tx = threadIdx.x + 1;"),
])
def test_other_kernels_do_not_match(edit):
    src = patterns.C1_F32.replace(*edit)
    assert src != patterns.C1_F32
    assert patterns.match(_k(src)) is None


def test_inconsistent_renaming_rejected():
    # two template names mapped onto one kernel name: not a bijection
    src = patterns.C1_I32.replace("i32 tx = threadIdx.x;", "i32 sum2 = threadIdx.x;") \
        .replace("tx", "sum2")
    assert patterns.match(_k(src)) is not None  # consistent rename: fine
    src = patterns.C1_I32.replace("tx / 32", "sum / 32")
    assert patterns.match(_k(src)) is None


def test_corpus_and_pins_route_generic():
    for f in ("C4_COMPACT_SERIAL", "C5_HIST_PER_BIN"):
        assert patterns.match(_k((GOLDEN / f"{f}.spk").read_text())) is None
