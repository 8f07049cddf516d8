"""paper_2112_10034_b200 — B200-native warp-primitive kernels behind the
warpfold launch API (arXiv 2112.10034, COX hierarchical collapsing).

The reference runs CUDA-style SPMD kernels on CPU threads by collapsing warps
and blocks into loop nests.  This package runs the same data-parallel path
natively on sm_100a: SHFL / VOTE / REDUX do the warp work, persistent grids
stream HBM with 16-byte loads, scans and compaction use decoupled look-back,
and the byte histogram is privatised in shared memory.  The public surface
mirrors the reference (``LaunchConfig``, ``DeviceMemory``, ``launch``, the
exception classes) and adds tensor-level ops.
"""

from .config import LaunchConfig
from .errors import (BarrierViolation, ConfigError, DivergenceError, ExecutionError,
                     LaunchError, NativeLibraryMissing, ParseError, SemanticError,
                     TransformError, UnsupportedFeatureError, WarpfoldError)

__version__ = "0.1.0"

_LAZY = {
    "DeviceMemory": ("memory", "DeviceMemory"),
    "launch": ("runtime", "launch"),
    "bind_args": ("runtime", "bind_args"),
    "PROGRAMS": ("runtime", "PROGRAMS"),
    "warp_program": ("runtime", "warp_program"),
    "ops": ("ops", None),
    "distributed": ("distributed", None),
    "dsl": ("dsl", None),
    "parse_module": ("dsl", "parse_module"),
    "hybrid_transform": ("dsl", "hybrid_transform"),
    "ExecTrace": ("trace", "ExecTrace"),
}


def __getattr__(name):
    # torch-dependent modules load lazily so the config/errors layer (and the
    # CPU-only tests) import without initialising CUDA
    if name in _LAZY:
        import importlib
        mod_name, attr = _LAZY[name]
        mod = importlib.import_module(f".{mod_name}", __name__)
        return mod if attr is None else getattr(mod, attr)
    raise AttributeError(name)


__all__ = ["LaunchConfig", "DeviceMemory", "launch", "ExecTrace", "bind_args", "PROGRAMS", "warp_program",
           "ops", "distributed", "parse_module", "hybrid_transform", "WarpfoldError",
           "ParseError", "SemanticError", "UnsupportedFeatureError", "TransformError",
           "ConfigError", "LaunchError", "ExecutionError", "BarrierViolation",
           "DivergenceError", "NativeLibraryMissing", "__version__"]
