"""The warpfold kernel language on B200: parse (reference dsl/), check, and
compile straight to sm_100a (replacing passes/ + interp/mpmd.py)."""

from .checker import SymbolTable, check_kernel
from .codegen import generate
from .jit import JitProgram, TransformOptions, hybrid_transform, resolve_mode, specialize
from .nodes import KernelDef, KernelModule, uses_warp_features
from .parser import parse_module, tokenize

__all__ = ["SymbolTable", "check_kernel", "generate", "JitProgram", "TransformOptions",
           "hybrid_transform", "resolve_mode", "specialize", "KernelDef", "KernelModule",
           "uses_warp_features", "parse_module", "tokenize"]
