"""Host-description programs (reference runtime/hostdesc.py, docs/hostdesc.md)
executed on the GPU, and the CLI `run` command."""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")

from oracle import numpy_oracle as no  # noqa: E402

DATA = Path(__file__).resolve().parent / "data"


@pytest.fixture(scope="module")
def built():
    from paper_2112_10034_b200 import build
    build.build_library()


def _expected():
    a = (-100 + 3 * np.arange(256)).astype(np.int32)
    p = np.concatenate([no.scan_inclusive_i32(s) for s in a.reshape(-1, 32)])
    g = no.scan_inclusive_i32(a * 2)
    u = (7 * np.arange(1000)).astype(np.uint8)
    return p, g, no.histogram256_u8(u)


def test_run_description(built):
    from paper_2112_10034_b200 import LaunchConfig
    from paper_2112_10034_b200.hostdesc import run_description
    _, dumps = run_description(DATA / "scan_pipeline.json", LaunchConfig())
    p, g, bins = _expected()
    assert [d["buffer"] for d in dumps] == ["p", "g", "bins"]
    assert dumps[0]["values"] == p.tolist()
    assert dumps[1]["values"] == g.tolist()
    assert dumps[2]["values"] == bins.astype(int).tolist()


def test_cli_run_json_and_errors(built, capsys, tmp_path):
    from paper_2112_10034_b200.__main__ import main
    assert main(["run", str(DATA / "scan_pipeline.json"), "--json"]) == 0
    lines = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert lines[1]["values"] == _expected()[1].tolist()
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"kernel_file": str(DATA / "scan_pipeline.spk"),
                               "buffers": [{"name": "a", "count": 4}],
                               "steps": [{"op": "launch", "kernel": "scale", "block": 32,
                                          "args": ["a", 2]}]}))
    assert main(["run", str(bad)]) == 4  # out-of-bounds -> EXIT_RUNTIME
    # the right-hand side a[tid] is evaluated before the store, like the
    # reference; thread 4 (lowest faulting id) reports
    assert "out-of-bounds read a[4], length 4" in capsys.readouterr().err
    assert main(["run", str(tmp_path / "missing.json")]) == 2


def test_cli_run_trace_counts(built, tmp_path):
    # cli.py:90-94: --trace-counts writes ExecTrace.to_json() of the DSL launches
    from paper_2112_10034_b200.__main__ import main
    out = tmp_path / "counts.json"
    assert main(["run", str(DATA / "scan_pipeline.json"), "--trace-counts", str(out)]) == 0
    data = json.loads(out.read_text())
    assert set(data) >= {"instructions", "terminators"}
    assert data["instructions"] and all(v > 0 for v in data["instructions"].values())
    # uid 1 is every DSL kernel's exit Ret: reached once per launched thread
    assert data["terminators"]["1"] % 32 == 0
