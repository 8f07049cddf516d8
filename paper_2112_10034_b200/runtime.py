"""``launch(program, config, memory, args)`` — the drop-in for the reference's
``warpfold.runtime.launch.launch`` (runtime/launch.py:90).

Reference flow: validate the config, return on an empty grid, bind and check
arguments (``bind_args``, runtime/launch.py:28-46), then run every block on
CPU workers and join.  Here the same validation and argument checks run in
Python (same messages), then the program's native entry point is enqueued on
the device and the call synchronises before returning — the reference's
join semantics (runtime/launch.py:1-8).  Programs are either

* ``NativeProgram`` objects for the five warp-primitive kernels and the warp
  collectives (``PROGRAMS`` below), or
* DSL kernels compiled to sm_100a by ``paper_2112_10034_b200.dsl`` (the
  ``hybrid_transform`` analogue).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import ops
from .config import LaunchConfig
from .errors import ConfigError, ExecutionError, LaunchError, UnsupportedFeatureError
from .memory import DeviceMemory


@dataclass(frozen=True)
class Param:
    name: str
    kind: str          # i32 | f32 | u8 | u64 | i64
    is_buffer: bool


@dataclass(eq=False)
class NativeProgram:
    """A launchable program backed by a native sm_100a entry point."""
    name: str
    params: list
    run: Callable = field(repr=False)
    mode: str = "hier"
    warp_size: int = 32
    # program-level grid: "op" = the op sizes its own persistent grid from n;
    # "spmd" = one logical thread per grid*block (the reference's model)
    grid_model: str = "op"


def _is_int(a) -> bool:
    return isinstance(a, (int, np.integer)) and not isinstance(a, bool)


def bind_args(params, memory: DeviceMemory, args) -> dict:
    """Check arity/kinds and resolve buffer ids to typed device views
    (same checks and messages as runtime/launch.py:28-46)."""
    if len(params) != len(args):
        raise LaunchError(f"kernel takes {len(params)} arguments, got {len(args)}")
    bound = {}
    for p, a in zip(params, args):
        if p.is_buffer:
            if not _is_int(a):
                raise LaunchError(f"argument {p.name!r} must be a buffer id, got {a!r}")
            bound[p.name] = memory.bind_view(int(a), p.kind)
        elif p.kind in ("i32", "i64"):
            if not _is_int(a):
                raise LaunchError(f"argument {p.name!r} must be an {p.kind} scalar, got {a!r}")
            bound[p.name] = int(a)
        else:
            if isinstance(a, bool) or not isinstance(a, (int, float, np.floating, np.integer)):
                raise LaunchError(f"argument {p.name!r} must be an f32 scalar, got {a!r}")
            bound[p.name] = np.float32(a)
    return bound


def launch(program, config: LaunchConfig, memory: DeviceMemory, args, trace=None) -> None:
    config.validate(hierarchical=(getattr(program, "mode", "hier") == "hier"))
    if config.device is not None and int(config.device) != memory.device.index:
        # the buffers live on the memory's device; a launch elsewhere would
        # read them over the peer path or fault
        raise ConfigError(f"LaunchConfig.device is {config.device} but the memory's buffers "
                          f"live on cuda:{memory.device.index}")
    if config.grid_size == 0:
        return
    if trace is not None and isinstance(program, NativeProgram):
        raise UnsupportedFeatureError(
            f"execution-count tracing (ExecTrace) needs a DSL kernel; {program.name!r} is a "
            f"named native op with no reference CFG")
    bound = bind_args(program.params, memory, args)
    with torch.cuda.device(memory.device):
        try:
            if trace is None:
                program.run(config, memory, bound)
            else:  # DSL kernel compiled with per-uid counters (interp/trace.py:9-50)
                program.run(config, memory, bound, trace=trace)
            torch.cuda.current_stream(memory.device).synchronize()
        finally:  # numpy views of the bound buffers show what the kernel wrote
            memory.refresh([int(a) for p, a in zip(program.params, args) if p.is_buffer])


# ---- named programs (K1-K5) ------------------------------------------------

def _span(bound: dict, name: str, n: int, access: str = "read"):
    t = bound[name]
    if n < 0:
        raise LaunchError(f"element count must be >= 0, got {n}")
    if n > t.numel():
        raise ExecutionError(
            f"out-of-bounds {access} {name}[{n - 1}], length {t.numel()}")
    return t[:n]


def _run_reduce_i32(config, memory, b):
    n = b["n"]
    a = _span(b, "a", n)
    out = _span(b, "out", 1, "write")
    ops.reduce_sum_i32(a, out, block=config.block_size if config.block_size in
                       ops.REDUCE_BLOCKS else 256)


def _run_reduce_f32(config, memory, b):
    n = b["n"]
    a = _span(b, "a", n)
    out = _span(b, "out", 1, "write")
    ops.reduce_sum_f32(a, out, block=config.block_size if config.block_size in
                       ops.REDUCE_BLOCKS else 256)


def _run_scan(config, memory, b):
    n = b["n"]
    ops.scan_inclusive_i32(_span(b, "a", n), _span(b, "out", n, "write"))


def _run_compact(config, memory, b):
    n = b["n"]
    ops.compact_gt0_i32(_span(b, "a", n), _span(b, "out", n, "write"),
                        _span(b, "count", 1, "write"))


def _run_hist(config, memory, b):
    n = b["n"]
    ops.histogram256_u8(_span(b, "a", n), _span(b, "bins", 256, "write"))


def _P(*spec):
    return [Param(*s) for s in spec]


PROGRAMS = {
    "reduce_sum_i32": NativeProgram(
        "reduce_sum_i32", _P(("a", "i32", True), ("out", "i32", True), ("n", "i64", False)),
        _run_reduce_i32),
    "reduce_sum_f32": NativeProgram(
        "reduce_sum_f32", _P(("a", "f32", True), ("out", "f32", True), ("n", "i64", False)),
        _run_reduce_f32),
    "scan_inclusive_i32": NativeProgram(
        "scan_inclusive_i32", _P(("a", "i32", True), ("out", "i32", True), ("n", "i64", False)),
        _run_scan),
    "compact_gt0_i32": NativeProgram(
        "compact_gt0_i32", _P(("a", "i32", True), ("out", "i32", True), ("count", "u64", True),
                              ("n", "i64", False)),
        _run_compact),
    "histogram256_u8": NativeProgram(
        "histogram256_u8", _P(("a", "u8", True), ("bins", "u64", True), ("n", "i64", False)),
        _run_hist),
}


def warp_program(kind: str, mask: int = 0xFFFFFFFF, per_lane_operand: bool = True,
                 operand: int = 0) -> NativeProgram:
    """SPMD program ``out[tid] = <kind>(a[tid], b[tid])`` over grid*block
    threads with warp width ``config.warp_size`` — the native form of the
    reference's collective semantics (interp/oracle.py:147-161)."""

    def run(config, memory, b):
        n = config.grid_size * config.block_size
        a = _span(b, "a", n)
        off = _span(b, "b", n) if per_lane_operand else None
        out = _span(b, "out", n, "write")
        ops.warp_collective(kind, a, off, operand=operand, block=config.block_size,
                            width=config.warp_size, mask=mask, out=out)

    params = [("a", "i32", True)] + ([("b", "i32", True)] if per_lane_operand else []) + [
        ("out", "i32", True)]
    return NativeProgram(f"warp_{kind}", _P(*params), run, grid_model="spmd")
