"""Checker-only access to the reference implementation (``warpfold``) for the
``diff`` command — never imported by a kernel or op path.

The reference is pure Python; it is importable when it is on ``sys.path``
already, installed under ``baseline/_ref`` (the offline install the bench
contract describes), or pointed to by ``$WARPFOLD_REF`` (a directory holding
the ``warpfold`` package).  Its own host-description runner executes the
description with ``engine="oracle"`` (runtime/hostdesc.py:97-129 ->
interp/oracle.py ``run_oracle``), exactly what the reference's ``diff``
compares against (cli.py:105-125)."""

from __future__ import annotations

import importlib
import os
import sys
from pathlib import Path

from .errors import UnsupportedFeatureError

ROOT = Path(__file__).resolve().parents[1]


def import_reference():
    """The ``warpfold`` package, or UnsupportedFeatureError saying where it
    was looked for."""
    try:
        return importlib.import_module("warpfold")
    except ImportError:
        pass
    for cand in (os.environ.get("WARPFOLD_REF"), str(ROOT / "baseline" / "_ref")):
        if cand and (Path(cand) / "warpfold" / "__init__.py").is_file():
            if cand not in sys.path:
                sys.path.append(cand)
            return importlib.import_module("warpfold")
    raise UnsupportedFeatureError(
        "the reference implementation (warpfold) is not importable: install it under "
        "baseline/_ref, set WARPFOLD_REF, or diff against committed dumps (--expected)")


def run_reference(description, kernel_path: str | None, config) -> tuple[dict, dict, list]:
    """Run the description through the reference's own oracle engine.
    Returns (buffer id -> final bytes, buffer id -> kind, dump payloads)."""
    import_reference()
    from warpfold.config import LaunchConfig as RefConfig
    from warpfold.runtime.hostdesc import HostProgram, load_description
    desc = load_description(description)
    host = HostProgram(desc, Path(description).parent, kernel_path)
    cfg = RefConfig(grid_size=config.grid_size, block_size=config.block_size,
                    warp_size=config.warp_size, mode=config.mode,
                    specialize=config.specialize, workers=1)
    dumps = host.run(cfg, engine="oracle")
    final = {bid: host.memory.copy_out(bid) for bid, _, _ in host.buffers.values()}
    kinds = {bid: kind for bid, kind, _ in host.buffers.values()}
    return final, kinds, dumps
