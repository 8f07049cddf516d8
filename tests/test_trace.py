"""ExecTrace parity: DSL kernels compiled in trace mode count every executed
instruction and terminator once per thread under the reference's own uids
(interp/trace.py:9-50, counted as interp/oracle.py:113-136 counts them) —
the GPU analogue of the reference's tests/test_counts.py:13-84.

CPU tests pin the uid numbering against the reference's CFG builder
(cfg/build.py, catalogue in tests/golden/corpus_traces.json); GPU tests
compare the device counts with run_oracle's ExecTrace for the whole corpus."""

import json
from pathlib import Path

import pytest

from paper_2112_10034_b200.dsl import parse_module
from paper_2112_10034_b200.dsl.checker import check_kernel
from paper_2112_10034_b200.dsl.codegen import generate, generate_traced
from paper_2112_10034_b200.trace import ExecTrace

GOLDEN = Path(__file__).resolve().parent / "golden"
TRACES = json.loads((GOLDEN / "corpus_traces.json").read_text())
MANIFEST = json.loads((GOLDEN / "corpus_manifest.json").read_text())


def _sources() -> dict:
    src = {m["kernel"]: m["source"] for m in MANIFEST.values()}
    for name in ("C1_I32", "C1_F32", "C3_WARP_PREFIX"):
        src[name] = (GOLDEN / f"{name}.spk").read_text()
    return src


SOURCES = _sources()


@pytest.mark.parametrize("name", sorted(TRACES["kernels"]))
def test_uid_numbering_matches_reference_cfg_builder(name):
    k = parse_module(SOURCES[name]).kernel()
    _, _, layout = generate_traced(k, check_kernel(k))
    want = TRACES["kernels"][name]
    assert {str(u): c for u, c in layout.kinds.items()} == want["uid_kinds"]
    assert layout.max_uid == want["max_uid"]


@pytest.mark.parametrize("name", sorted(TRACES["kernels"]))
def test_traced_source_differs_only_by_counters(name):
    k = parse_module(SOURCES[name]).kernel()
    t = check_kernel(k)
    plain, _ = generate(k, t)
    traced, _, layout = generate_traced(k, t)
    assert "wf_tick" not in plain.split("wf_kernel", 1)[1]
    assert traced.count("wf_tick(wf_tr,") >= len(layout.instr_uids)


def test_exec_trace_api_mirrors_reference():
    a, b = ExecTrace(), ExecTrace()
    a.count_instr(3)
    a.count_instr(3, 4)
    b.count_instr(3)
    b.count_term(7, 2)
    b.record_arrival(9, [0, 1])
    m = a.merged(b)
    assert m.instr_counts[3] == 6 and m.term_counts[7] == 2
    assert m.counts_by_src({3: 1}) == {1: 6}
    j = m.to_json({})
    assert j["instructions"] == {"3": 6} and j["terminators"] == {"7": 2}
    assert j["barrier_arrivals"] == {"9": [[0, 1]]}
    assert a.instr_counts[3] == 5  # merged() does not mutate its inputs


@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted(TRACES["runs"]))
def test_gpu_exec_counts_equal_reference_oracle(tag):
    torch = pytest.importorskip("torch")
    import numpy as np

    import paper_2112_10034_b200 as wf
    from paper_2112_10034_b200.dsl import hybrid_transform

    m = MANIFEST[tag]
    arrays = np.load(GOLDEN / "corpus.npz")
    kernel = parse_module(m["source"]).kernel()
    mem = wf.DeviceMemory()
    ids = []
    for i, kind in enumerate(m["kinds"]):
        init = arrays[f"{tag}__in{i}"]
        b = mem.alloc(4 * len(init))
        mem.write(b, init, kind)
        ids.append(b)
    it = iter(ids)
    scalars = iter(a[1] for a in m["args"] if a[0] == "scalar")
    args = [next(it) if p.is_buffer else next(scalars) for p in kernel.params]
    cfg = wf.LaunchConfig(grid_size=m["grid"], block_size=m["block"], warp_size=m["warp"])
    prog = hybrid_transform(kernel, cfg)
    trace = ExecTrace()
    wf.launch(prog, cfg, mem, args, trace=trace)
    torch.cuda.synchronize()
    want = TRACES["runs"][tag]
    max_uid = TRACES["kernels"][m["kernel"]]["max_uid"]
    for uid in prog.original_instr_uids:
        assert trace.instr_counts.get(uid, 0) == want["instr"].get(str(uid), 0), (tag, uid)
    assert {str(u) for u in trace.instr_counts} == set(want["instr"])
    for uid in prog.layout.term_uids:
        assert trace.term_counts.get(uid, 0) == want["term"].get(str(uid), 0), (tag, uid)
    # the oracle's only other terminators are blocks canonicalize() inserted
    extra = {int(u) for u in want["term"]} - set(prog.layout.term_uids)
    assert all(u > max_uid for u in extra), (tag, extra)
    # every thread reaches the exit exactly once (the Ret allocated first)
    assert trace.term_counts[1] == m["grid"] * m["block"]
    # barrier arrival sets, episode by episode in the oracle's order
    # (interp/oracle.py:207 warp barriers, :237 block barriers)
    got = {str(u): [sorted(s) for s in sets] for u, sets in trace.barrier_arrivals.items()}
    assert got == want.get("arrivals", {}), tag
