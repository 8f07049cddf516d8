"""Structural registry: the reference's own DSL formulations of the hot path
-> native sm_100a kernels ("dispatches via a registry (DSL AST
or op name -> native symbol)").

The reference can write C1/C2 only as the per-warp-partials kernel of
SURVEY §8c and C3 only as the in-warp prefix on lane-reversed data; its
users reach them through ``launch(hybrid_transform(kernel, cfg), ...)``
(runtime/launch.py:90, passes/pipeline.py:103-179).  ``match`` recognises
those kernels up to renaming (kernel, parameter and local names; any
alpha-equivalent spelling of the same AST) and returns a ``NativePattern``;
``JitProgram.run`` then calls its C-ABI kernel (``csrc/wf_patterns.cu``)
instead of the generic codegen.  The native kernels write exactly what the
DSL kernel writes — fp32 partials in the reference's association included —
whenever ``applicable`` holds; otherwise (other warp size, buffers too short,
aliasing, i32 index wrap) the generic compiled kernel runs, so faults and
wrap-around keep the DSL's behaviour.  Both paths are native GPU code.

Templates are the kernels the reference itself runs for this path
(tests/golden/make_golden.py, pinned by tests/golden/c1c2_pin.npz and
c3_pin.npz).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

from . import nodes as n

C1_I32 = """
__global__ void wsum(global i32* a, global i32* out, i32 n) {
    i32 tx = threadIdx.x;
    i32 sum = 0;
    for (i32 i = tx + blockIdx.x * blockDim.x; i < n; i = i + blockDim.x * gridDim.x) {
        sum = sum + a[i];
    }
    for (i32 off = 16; off > 0; off = off / 2) {
        sum = sum + shfl_down(sum, off);
    }
    if (tx % 32 == 0) {
        out[blockIdx.x * (blockDim.x / 32) + tx / 32] = sum;
    }
}
"""
C1_F32 = C1_I32.replace("global i32* a, global i32* out", "global f32* a, global f32* out") \
               .replace("i32 sum = 0;", "f32 sum = 0.0;")

C3_WARP_PREFIX = """
__global__ void warp_prefix(global i32* a, global i32* out) {
    i32 tid = threadIdx.x + blockIdx.x * blockDim.x;
    i32 lane = threadIdx.x % 32;
    i32 base = tid - lane;
    i32 v = a[base + 31 - lane];
    for (i32 off = 1; off < 32; off = off * 2) {
        i32 t = shfl_down(v, off);
        if (lane + off < 32) {
            v = v + t;
        }
    }
    out[base + 31 - lane] = v;
}
"""

# dataclass fields that hold identifiers (renamable); everything else must match exactly
_NAME_FIELDS = {
    (n.Param, "name"), (n.VarRef, "name"), (n.VarTarget, "name"), (n.IndexExpr, "base"),
    (n.IndexTarget, "base"), (n.DeclLocal, "name"), (n.DeclShared, "name"),
}
I32_MAX = (1 << 31) - 1


def _alpha_eq(a, b, fwd: dict, back: dict) -> bool:
    """Structural equality up to a consistent bijective renaming."""
    if type(a) is not type(b):
        return False
    if isinstance(a, (tuple, list)):
        return len(a) == len(b) and all(_alpha_eq(x, y, fwd, back) for x, y in zip(a, b))
    if dataclasses.is_dataclass(a):
        for f in dataclasses.fields(a):
            x, y = getattr(a, f.name), getattr(b, f.name)
            if (type(a), f.name) in _NAME_FIELDS:
                if fwd.setdefault(x, y) != y or back.setdefault(y, x) != x:
                    return False
            elif not _alpha_eq(x, y, fwd, back):
                return False
        return True
    return a == b


@dataclass(frozen=True)
class NativePattern:
    """A recognised reference formulation and the native kernel that runs it."""
    name: str          # warp_partials_sum_i32 | warp_partials_sum_f32 | warp_prefix32_i32
    symbol: str        # C-ABI entry point (include/warpfold_b200.h)
    a: str             # the kernel's own parameter names, by role
    out: str
    n: str | None = None

    def applicable(self, config, bound: dict) -> bool:
        """True iff the native kernel writes exactly what the DSL kernel would,
        with no fault: warp 32, no i32 index wrap, every access in bounds,
        distinct buffers."""
        if config.warp_size != 32 or config.block_size % 32:
            return False
        a, out = bound[self.a], bound[self.out]
        if _overlap(a, out):
            return False
        threads = config.grid_size * config.block_size
        if self.n is None:  # warp prefix: thread t reads and writes element t
            return threads <= I32_MAX and a.numel() >= threads and out.numel() >= threads
        nv = int(bound[self.n])
        return (threads + max(nv, 0) <= I32_MAX and a.numel() >= max(nv, 0)
                and out.numel() >= threads // 32)

    def run(self, config, bound: dict, stream: int) -> None:
        from .. import _lib
        lib = _lib.load()
        a, out = bound[self.a], bound[self.out]
        if self.n is None:
            rc = lib.wf_warp_prefix32_i32(a.data_ptr(), out.data_ptr(),
                                          config.grid_size * config.block_size, stream)
        else:
            rc = getattr(lib, self.symbol)(a.data_ptr(), int(bound[self.n]), out.data_ptr(),
                                           config.grid_size, config.block_size, stream)
        _lib.check(rc, self.symbol)


def _overlap(x, y) -> bool:
    xs, ys = x.data_ptr(), y.data_ptr()
    xe, ye = xs + x.numel() * x.element_size(), ys + y.numel() * y.element_size()
    return xs < ye and ys < xe


_TEMPLATES = None


def _templates():
    global _TEMPLATES
    if _TEMPLATES is None:
        from .parser import parse_module
        _TEMPLATES = [
            ("warp_partials_sum_i32", "wf_warp_partials_sum_i32",
             parse_module(C1_I32).kernel()),
            ("warp_partials_sum_f32", "wf_warp_partials_sum_f32",
             parse_module(C1_F32).kernel()),
            ("warp_prefix32_i32", "wf_warp_prefix32_i32", parse_module(C3_WARP_PREFIX).kernel()),
        ]
    return _TEMPLATES


def match(kernel: n.KernelDef) -> NativePattern | None:
    """The native pattern ``kernel`` is an alpha-renaming of, or None."""
    for name, symbol, tmpl in _templates():
        fwd, back = {}, {}
        if _alpha_eq(tmpl.params, kernel.params, fwd, back) and \
                _alpha_eq(tmpl.body, kernel.body, fwd, back):
            return NativePattern(name, symbol, a=fwd["a"], out=fwd["out"],
                                 n=fwd.get("n") if name != "warp_prefix32_i32" else None)
    return None
