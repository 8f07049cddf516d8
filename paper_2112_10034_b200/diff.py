"""Differential comparison of a GPU run against a reference run — the
reference's ``interp/diff.py:19-91`` (``DiffReport``, ``compare_memory`` with
an absolute ``fp_tol`` on f32 buffers) and the ``diff`` CLI command
(cli.py:105-125).

Two reference sides are supported:

* the reference interpreter itself (``warpfold``'s ``run_oracle`` through its
  own ``HostProgram(..., engine="oracle")``), when that package is importable
  — run by the checker-only module :mod:`.refcheck`, never by a kernel path;
* committed expected dumps (the JSON lines ``warpfold run desc.json --json``
  prints), so a GPU box without the reference installed can still diff.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np

from .memory import numpy_dtype


@dataclass
class DiffReport:
    """interp/diff.py:19-29: equal flag, human detail, first divergence."""
    equal: bool
    detail: str = "equal"
    divergence: Optional[dict] = field(default=None)

    def to_json(self) -> dict:
        data = {"equal": self.equal, "detail": self.detail}
        if self.divergence:
            data["divergence"] = self.divergence
        return data


def _first_divergence(buffer, kind: str | None, ref: bytes, got: bytes) -> dict:
    """First differing element (typed when the kind is known, else byte)."""
    if kind is not None and len(ref) == len(got):
        dt = numpy_dtype(kind)
        item = np.dtype(dt).itemsize
        a = np.frombuffer(ref[:len(ref) - len(ref) % item], dtype=dt)
        b = np.frombuffer(got[:len(got) - len(got) % item], dtype=dt)
        bad = np.nonzero(a.view(f"u{item}") != b.view(f"u{item}"))[0]
        if len(bad):
            i = int(bad[0])
            conv = float if kind == "f32" else int
            return {"buffer": buffer, "element": i, "reference": conv(a[i]),
                    "transformed": conv(b[i])}
    for i, (x, y) in enumerate(zip(ref, got)):
        if x != y:
            return {"buffer": buffer, "byte": i, "reference": x, "transformed": y}
    return {"buffer": buffer, "byte": min(len(ref), len(got)), "detail": "length mismatch"}


def _report(div: dict) -> DiffReport:
    where = f"element {div['element']}" if "element" in div else f"byte {div.get('byte')}"
    return DiffReport(False, f"buffer {div['buffer']} diverges at {where}: "
                             f"reference={div.get('reference')} "
                             f"transformed={div.get('transformed')}", div)


def _fp_close(ref: bytes, got: bytes, fp_tol: float) -> bool:
    a = np.frombuffer(ref, dtype=np.float32)
    b = np.frombuffer(got, dtype=np.float32)
    return bool(np.allclose(a, b, rtol=0.0, atol=fp_tol, equal_nan=True))


def compare_memory(reference: dict, transformed: dict, buffer_kinds: dict | None = None,
                   fp_tol: float = 0.0) -> DiffReport:
    """``reference`` / ``transformed``: buffer id -> bytes.  Same order, kinds
    and tolerance rule as interp/diff.py:48-72 (bit-exact unless an f32
    buffer is within the absolute ``fp_tol``)."""
    buffer_kinds = buffer_kinds or {}
    for bid in sorted(set(reference) | set(transformed)):
        ref, got = reference.get(bid, b""), transformed.get(bid, b"")
        if ref == got:
            continue
        kind = buffer_kinds.get(bid)
        if fp_tol > 0.0 and kind == "f32" and len(ref) == len(got) and _fp_close(ref, got, fp_tol):
            continue
        return _report(_first_divergence(bid, kind, ref, got))
    return DiffReport(True)


def _payload_bytes(p: dict) -> bytes:
    return np.asarray(p["values"], dtype=numpy_dtype(p["kind"])).tobytes()


def compare_dumps(expected: list, got: list, fp_tol: float = 0.0) -> DiffReport:
    """Dump payloads ({"buffer", "kind", "values"}) in step order."""
    if [p["buffer"] for p in expected] != [p["buffer"] for p in got]:
        return DiffReport(False, f"dumped buffers differ: reference "
                                 f"{[p['buffer'] for p in expected]} vs transformed "
                                 f"{[p['buffer'] for p in got]}")
    for e, g in zip(expected, got):
        ref, out = _payload_bytes(e), _payload_bytes(g)
        if ref == out:
            continue
        if fp_tol > 0.0 and e["kind"] == "f32" and len(ref) == len(out) and \
                _fp_close(ref, out, fp_tol):
            continue
        return _report(_first_divergence(e["buffer"], e["kind"], ref, out))
    return DiffReport(True)


def load_dumps(path) -> list:
    """Expected dumps: one JSON payload per line (``run --json`` output)."""
    lines = Path(path).read_text(encoding="utf-8").splitlines()
    return [json.loads(x) for x in lines if x.strip()]
