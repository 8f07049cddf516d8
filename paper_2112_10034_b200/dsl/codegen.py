"""DSL kernel -> CUDA C for sm_100a, with the reference's semantics.

Replaces the collapsing pipeline (passes/pipeline.py:103-179) and the MPMD
interpreter (interp/mpmd.py:237-255): the GPU runs the kernel as real SIMT
code, so instead of wrapping regions in lane/warp loops the generator only has
to make every scalar operation mean exactly what it means in the reference:

* i32 wraps mod 2^32 (numerics.py:20-22) -> unsigned arithmetic helpers;
  ``/`` and ``%`` truncate and fault on zero (numerics.py:25-37), including
  INT_MIN / -1 = INT_MIN.
* f32 is IEEE single, one rounding per op, no contraction ->
  ``__fadd_rn``/``__fmul_rn``/``__fdiv_rn`` and NVRTC ``--fmad=false``;
  i32 operands widen with round-to-nearest (np.float32(int)).
* ``&&``/``||`` evaluate both operands (interp/evalexpr.py:36-40), results
  are i32 0/1.
* Locals live in one flat per-kernel namespace and read as zero until
  assigned (interp/oracle.py:45-46): all are hoisted to the kernel top and
  zero-initialised; a declaration with an initializer becomes an assignment.
* Shared arrays are zero-filled per block (interp/oracle.py:214-216).
* Every global/shared access is bounds-checked; a violation records the
  reference's message ("out-of-bounds read a[100], length 32",
  interp/oracle.py:65-81) in a device error record, the access reads 0 / is
  dropped, the faulting thread leaves every loop at its next test (it stays
  alive, so warp collectives keep their participants), and the host raises
  ExecutionError after the launch.
* Step limit (interp/oracle.py:113-119): every loop iteration counts one
  step per thread; a thread past ``wf_step_limit`` records "thread T
  exceeded the step limit" and leaves its loops, so a non-terminating kernel
  ends with ExecutionError instead of hanging the GPU.  (An earlier form that
  `return`ed from inside the loop made NVRTC miscompile kernels that mix
  segment-masked votes with such loops: fuzz seeds 444 / 713 at W = 4.)
* Collectives follow passes/warp_lower.py:17-45 / interp/oracle.py:147-161:
  ``shfl_down`` hands out-of-range lanes their own value for ANY offset (one
  SHFL.IDX with an explicitly computed source lane, not the 5-bit-masked
  SHFL.DOWN), votes return 0/1.  The reference's warp of W lanes is a
  W-lane segment of the hardware warp (W = LaunchConfig.warp_size).

Trace mode (``trace=True``) adds execution counting with the reference's
instruction identities: uids are allocated in exactly the order
cfg/build.py:37-186 allocates them (exit ``Ret`` first, collectives hoisted
left to right before their statement, a guard and a latch ``CondBr`` per loop
with the condition's collectives lowered twice, nothing after a ``return``),
and every executed instruction / terminator bumps its counter once per thread,
as ``interp/oracle.py:113-136`` counts them.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from ..errors import TransformError
from . import nodes as n
from .checker import SymbolTable, expr_kind

I32, F32 = n.I32, n.F32
CTYPE = {I32: "int", F32: "float"}

PRELUDE = r"""
#define WF_INT_MIN (-2147483647 - 1)
struct wf_err_t {
  unsigned long long code; long long arg; long long index; long long length;
  unsigned long long key; unsigned int lock;
};
// Record a fault.  The fault of the lowest global thread id wins (keeps the
// message reproducible run to run); a thread keeps its first fault.  Faults
// are rare, so a short spin lock guards the record.
__device__ __noinline__ void wf_fail(wf_err_t *e, unsigned long long code, long long arg,
                                     long long idx, long long len) {
  const unsigned long long key =
      (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x + 1ull;
  while (atomicCAS(&e->lock, 0u, 1u) != 0u) { __nanosleep(32); }
  __threadfence();
  if (e->key == 0ull || key < e->key) {
    e->key = key; e->code = code; e->arg = arg; e->index = idx; e->length = len;
  }
  __threadfence();
  atomicExch(&e->lock, 0u);
}
// execution counting (ExecTrace): one counter per reference CFG uid
__device__ __forceinline__ void wf_tick(unsigned long long *t, int uid) { atomicAdd(t + uid, 1ull); }
// barrier arrival log (ExecTrace.barrier_arrivals, interp/oracle.py:207,237):
// a[0] = record count; record i at a[4 + 4 i] = {uid, block, phase << 32 |
// warp episode, warp << 32 | arrival mask (warp = 0xffffffff: the whole block)}
__device__ __noinline__ void wf_arrive(unsigned long long *a, long long cap, int uid,
                                       unsigned long long ph_ep, unsigned long long warp_mask) {
  const unsigned long long i = atomicAdd(a, 1ull);
  if ((long long)i < cap) {
    unsigned long long *r = a + 4 + 4 * i;
    r[0] = (unsigned long long)uid; r[1] = blockIdx.x; r[2] = ph_ep; r[3] = warp_mask;
  }
}
__device__ __forceinline__ int wf_add(int a, int b) { return (int)((unsigned)a + (unsigned)b); }
__device__ __forceinline__ int wf_sub(int a, int b) { return (int)((unsigned)a - (unsigned)b); }
__device__ __forceinline__ int wf_mul(int a, int b) { return (int)((unsigned)a * (unsigned)b); }
__device__ __forceinline__ int wf_neg(int a) { return (int)(0u - (unsigned)a); }
// loop test: false once the thread faulted or ran out of steps
__device__ __forceinline__ bool wf_live(int &dead, long long &steps, long long limit, wf_err_t *e) {
  if (dead) return false;
  if (++steps > limit) {
    wf_fail(e, 5, -1, (long long)blockIdx.x * blockDim.x + threadIdx.x, 0);
    dead = 1;
    return false;
  }
  return true;
}
__device__ __forceinline__ int wf_div(int a, int b, wf_err_t *e, int &dead) {
  if (b == 0) { if (!dead) wf_fail(e, 3, -1, 0, 0); dead = 1; return 0; }
  if (a == WF_INT_MIN && b == -1) return WF_INT_MIN;
  return a / b;
}
__device__ __forceinline__ int wf_rem(int a, int b, wf_err_t *e, int &dead) {
  if (b == 0) { if (!dead) wf_fail(e, 4, -1, 0, 0); dead = 1; return 0; }
  if (b == -1) return 0;
  return a % b;
}
__device__ __forceinline__ float wf_f(int a) { return __int2float_rn(a); }
__device__ __forceinline__ float wf_f(float a) { return a; }
__device__ __forceinline__ int wf_land(int a, int b) { return (a != 0 && b != 0) ? 1 : 0; }
__device__ __forceinline__ int wf_lor(int a, int b) { return (a != 0 || b != 0) ? 1 : 0; }
template <typename T>
__device__ __forceinline__ T wf_ld(const T *p, long long len, long long i, long long arg, wf_err_t *e,
                                   int &dead) {
  if (i < 0 || i >= len) { if (!dead) wf_fail(e, 1, arg, i, len); dead = 1; return (T)0; }
  return p[i];
}
template <typename T>
__device__ __forceinline__ void wf_st(T *p, long long len, long long i, T v, long long arg, wf_err_t *e,
                                      int &dead) {
  if (i < 0 || i >= len) { if (!dead) wf_fail(e, 2, arg, i, len); dead = 1; return; }
  p[i] = v;
}
// ---- warp collectives over W-lane segments of the hardware warp ----------
__device__ __forceinline__ unsigned wf_present() {
  const unsigned k = blockDim.x - (threadIdx.x & ~31u);
  return k >= 32u ? 0xffffffffu : ((1u << k) - 1u);
}
__device__ __forceinline__ unsigned wf_seg() { return (threadIdx.x & 31u) & ~(WF_W - 1u); }
__device__ __forceinline__ unsigned wf_segbits() {
  return WF_W == 32 ? 0xffffffffu : (((1u << WF_W) - 1u) << wf_seg());
}
template <typename T>
__device__ __forceinline__ T wf_shfl_from(T v, long long src_in_seg, unsigned mask) {
  const unsigned lane = threadIdx.x & 31u;
  unsigned src = lane;
  if (src_in_seg >= 0 && src_in_seg < WF_W) {
    const unsigned s = wf_seg() + (unsigned)src_in_seg;
    if ((mask >> s) & 1u) src = s;
  }
  return __shfl_sync(mask, v, src);
}
__device__ __forceinline__ long long wf_lane_in_seg() { return (long long)((threadIdx.x & 31u) - wf_seg()); }
template <typename T> __device__ __forceinline__ T wf_shfl_down(T v, int off, unsigned m) {
  return wf_shfl_from(v, wf_lane_in_seg() + off, m); }
template <typename T> __device__ __forceinline__ T wf_shfl_up(T v, int off, unsigned m) {
  return wf_shfl_from(v, wf_lane_in_seg() - off, m); }
template <typename T> __device__ __forceinline__ T wf_shfl_xor(T v, int x, unsigned m) {
  return wf_shfl_from(v, (long long)((unsigned)wf_lane_in_seg() ^ (unsigned)x), m); }
template <typename T> __device__ __forceinline__ T wf_shfl_idx(T v, int s, unsigned m) {
  long long r = (long long)s % WF_W; if (r < 0) r += WF_W; return wf_shfl_from(v, r, m); }
__device__ __forceinline__ int wf_vote_all(int p, unsigned m) {
  const unsigned part = m & wf_segbits();
  return (__ballot_sync(m, p != 0) & part) == part ? 1 : 0; }
__device__ __forceinline__ int wf_vote_any(int p, unsigned m) {
  return (__ballot_sync(m, p != 0) & m & wf_segbits()) != 0u ? 1 : 0; }
__device__ __forceinline__ int wf_ballot(int p, unsigned m) {
  return (int)((__ballot_sync(m, p != 0) & m & wf_segbits()) >> wf_seg()); }
__device__ __forceinline__ int wf_reduce_add(int v, unsigned m) {
  if (WF_W == 32) return (int)__reduce_add_sync(m, (unsigned)v);
  unsigned acc = 0;
  for (unsigned j = 0; j < WF_W; ++j) {
    const unsigned s = wf_seg() + j;
    const bool ok = (m >> s) & 1u;
    const unsigned t = __shfl_sync(m, (unsigned)v, ok ? s : (threadIdx.x & 31u));
    acc += ok ? t : 0u;
  }
  return (int)acc;
}
"""

ERR_MESSAGES = {1: "read", 2: "write"}


def _f32_literal(v: float) -> str:
    bits = struct.unpack("<I", struct.pack("<f", float(np.float32(v))))[0]
    return f"__int_as_float(0x{bits:08x})"


def _i32_literal(v: int) -> str:
    v &= 0xFFFFFFFF
    return f"((int)0x{v:08x}u)"


class CudaGen:
    def __init__(self, kernel: n.KernelDef, table: SymbolTable, warp_size: int,
                 block_size: int | None = None, grid_size: int | None = None,
                 trace: bool = False):
        self.k, self.t, self.W = kernel, table, warp_size
        self.block_size, self.grid_size = block_size, grid_size  # specialize (JIT mode)
        self.trace = trace
        self.uid = 0                       # cfg/ir.py:154-161 (Cfg.new_uid)
        self.instr_uids: list[int] = []    # Assign / DeclLocal / DeclShared / Collective / Barrier
        self.term_uids: list[int] = []     # Br / CondBr / Ret allocated by the builder
        self.uid_kind: dict[int, str] = {}  # uid -> reference IR class name (cfg/ir.py)
        self.lines: list[str] = []
        self.arrays: list[str] = []  # error-record arg index -> array name
        for p in kernel.params:
            if p.is_buffer:
                self.arrays.append(p.name)
        for name in table.shared:
            self.arrays.append(name)

    # -- uids (trace mode)
    def new_uid(self, kind: str) -> int:
        self.uid += 1
        term = kind in ("Br", "CondBr", "Ret")
        (self.term_uids if term else self.instr_uids).append(self.uid)
        self.uid_kind[self.uid] = kind
        return self.uid

    def tick(self, uid: int) -> str:
        return f"wf_tick(wf_tr, {uid});" if self.trace else ""

    # -- names
    def arr_ptr(self, name: str) -> str:
        return f"p_{name}" if name in self.t.params else f"s_{name}"

    def arr_len(self, name: str) -> str:
        if name in self.t.params:
            return f"p_{name}_len"
        length = self.t.shared[name][1]
        return "wf_dyn_len" if length is None else f"{length}LL"

    def arr_id(self, name: str) -> int:
        return self.arrays.index(name)

    def var(self, name: str) -> str:
        return f"p_{name}" if name in self.t.params else f"v_{name}"

    # -- expressions -> (code, kind)
    def expr(self, e) -> tuple[str, str]:
        if isinstance(e, n.IntLit):
            return _i32_literal(e.value), I32
        if isinstance(e, n.FloatLit):
            return _f32_literal(e.value), F32
        if isinstance(e, n.VarRef):
            return self.var(e.name), expr_kind(e, self.t)
        if isinstance(e, n.BuiltinRef):
            if e.name == "blockDim.x" and self.block_size:
                return f"{self.block_size}", I32
            if e.name == "gridDim.x" and self.grid_size:
                return f"{self.grid_size}", I32
            return f"((int){e.name})", I32
        if isinstance(e, n.IndexExpr):
            idx, _ = self.expr(e.index)
            kind = self.t.element_kind(e.base)
            return (f"wf_ld<{CTYPE[kind]}>({self.arr_ptr(e.base)}, {self.arr_len(e.base)}, "
                    f"(long long)({idx}), {self.arr_id(e.base)}, wf_e, wf_dead)"), kind
        if isinstance(e, n.Unary):
            c, k = self.expr(e.operand)
            if e.op == "!":
                return f"(({c}) == 0 ? 1 : 0)", I32
            return (f"(-({c}))", F32) if k == F32 else (f"wf_neg({c})", I32)
        if isinstance(e, n.Binary):
            return self.binary(e)
        if isinstance(e, n.CollectiveCall):
            return self.collective(e)
        raise TransformError(f"cannot generate {type(e).__name__}")

    def binary(self, e: n.Binary) -> tuple[str, str]:
        a, ak = self.expr(e.left)
        b, bk = self.expr(e.right)
        if e.op == "&&":
            return f"wf_land({a}, {b})", I32
        if e.op == "||":
            return f"wf_lor({a}, {b})", I32
        f32 = F32 in (ak, bk)
        if e.op in ("==", "!=", "<", "<=", ">", ">="):
            if f32:
                a, b = f"wf_f({a})", f"wf_f({b})"
            return f"(({a}) {e.op} ({b}) ? 1 : 0)", I32
        if f32:
            fn = {"+": "__fadd_rn", "-": "__fsub_rn", "*": "__fmul_rn", "/": "__fdiv_rn"}[e.op]
            return f"{fn}(wf_f({a}), wf_f({b}))", F32
        if e.op in ("/", "%"):
            return f"{'wf_div' if e.op == '/' else 'wf_rem'}({a}, {b}, wf_e, wf_dead)", I32
        fn = {"+": "wf_add", "-": "wf_sub", "*": "wf_mul"}[e.op]
        return f"{fn}({a}, {b})", I32

    def mask(self, e) -> str:
        # a collective synchronises its LOGICAL warp only (the W-lane segment
        # of the hardware warp): at W < 32 one segment may execute it inside a
        # branch its neighbour skips (legal in the reference, whose aligned-
        # barrier rule is per logical warp), so the other segment's lanes must
        # not be named in the *_sync mask
        if e is None:
            return "(wf_present() & wf_segbits())"
        m, _ = self.expr(e)
        return f"((unsigned)({m}) & wf_present() & wf_segbits())"

    def collective(self, e: n.CollectiveCall) -> tuple[str, str]:
        # operands first, then the collective's own uid (cfg/build.py:153-159)
        if e.op in ("shfl_down", "shfl_up", "shfl_xor", "shfl_idx"):
            v, vk = self.expr(e.args[0])
            o, _ = self.expr(e.args[1])
            m = self.mask(e.mask)
            code, kind = f"wf_{e.op}<{CTYPE[vk]}>({v}, {o}, {m})", vk
        else:
            a, _ = self.expr(e.args[0])
            m = self.mask(e.mask)
            code, kind = f"wf_{e.op}({a}, {m})", I32
        uid = self.new_uid("Collective")
        if self.trace:
            code = f"(wf_tick(wf_tr, {uid}), {code})"
        return code, kind

    def convert(self, code: str, src: str, dst: str) -> str:
        return f"wf_f({code})" if (dst == F32 and src == I32) else code

    # -- statements
    def emit(self, line: str, depth: int):
        self.lines.append("  " * depth + line)

    def assign(self, s: n.Assign, depth: int, as_expr: bool = False) -> str:
        # store index, then value, then the Assign's uid (cfg/build.py:67-73)
        tg = s.target
        idx = self.expr(tg.index)[0] if isinstance(tg, n.IndexTarget) else None
        val, vk = self.expr(s.expr)
        uid = self.new_uid("Assign")
        if isinstance(tg, n.VarTarget):
            code = f"{self.var(tg.name)} = {self.convert(val, vk, self.t.locals[tg.name])}"
        else:
            kind = self.t.element_kind(tg.base)
            code = (f"wf_st<{CTYPE[kind]}>({self.arr_ptr(tg.base)}, {self.arr_len(tg.base)}, "
                    f"(long long)({idx}), {self.convert(val, vk, kind)}, {self.arr_id(tg.base)}, wf_e, "
                    f"wf_dead)")
        if self.trace:
            code = f"{code}, wf_tick(wf_tr, {uid})"
        if as_expr:
            return code
        self.emit(code + ";", depth)
        return code

    def stmts(self, body, depth: int) -> bool:
        """Returns False when control cannot fall through (after a return the
        reference lowers nothing more of the list, cfg/build.py:56-58)."""
        for s in body:
            if not self.stmt(s, depth):
                return False
        return True

    def decl_local(self, s: n.DeclLocal, depth: int) -> None:
        uid = self.new_uid("DeclLocal")
        if self.trace:
            self.emit(self.tick(uid), depth)
        if s.init is not None:
            v, vk = self.expr(s.init)
            a_uid = self.new_uid("Assign")
            self.emit(f"v_{s.name} = {self.convert(v, vk, s.kind)};{self.tick(a_uid)}", depth)

    def init_stmt(self, init, depth: int) -> None:
        if isinstance(init, n.DeclLocal):
            self.decl_local(init, depth)
        else:
            self.assign(init, depth)

    def stmt(self, s, depth: int) -> bool:
        if isinstance(s, n.DeclLocal):
            self.decl_local(s, depth)
        elif isinstance(s, n.DeclShared):
            uid = self.new_uid("DeclShared")  # storage hoisted; the declaration still executes
            if self.trace:
                self.emit(self.tick(uid), depth)
        elif isinstance(s, n.Assign):
            self.assign(s, depth)
        elif isinstance(s, n.If):
            c, _ = self.expr(s.cond)
            cb = self.new_uid("CondBr")
            self.emit(f"{self.tick(cb)}if (({c}) != 0) {{", depth)
            if s.then and self.stmts(s.then, depth + 1):
                self.emit(self.tick(self.new_uid("Br")), depth + 1)
            if s.orelse is not None:
                self.emit("} else {", depth)
                if s.orelse and self.stmts(s.orelse, depth + 1):
                    self.emit(self.tick(self.new_uid("Br")), depth + 1)
            self.emit("}", depth)
        elif isinstance(s, n.For):
            self.loop(s, depth)
        elif isinstance(s, n.SyncThreads):
            uid = self.new_uid("Barrier")
            if self.trace:  # one rendezvous of the whole block (interp/oracle.py:237)
                self.emit(f"{self.tick(uid)}if (threadIdx.x == 0) wf_arrive(wf_arr, wf_arr_cap, {uid}, "
                          f"(unsigned long long)wf_phase << 32, 0xffffffff00000000ull); "
                          f"__syncthreads(); ++wf_phase;", depth)
            else:
                self.emit("__syncthreads();", depth)
        elif isinstance(s, n.SyncWarp):
            m = self.mask(s.mask)
            uid = self.new_uid("Barrier")
            if self.trace:  # the logical warp's arriving lanes (interp/oracle.py:207)
                self.emit(f"{{ {self.tick(uid)}const unsigned wf_m = {m}; "
                          f"const unsigned wf_am = __activemask() & wf_m; "
                          f"if ((threadIdx.x & 31u) == (unsigned)(__ffs(wf_am) - 1)) "
                          f"wf_arrive(wf_arr, wf_arr_cap, {uid}, ((unsigned long long)wf_phase << 32) | "
                          f"(unsigned)wf_wep, ((unsigned long long)(threadIdx.x / WF_W) << 32) | "
                          f"(wf_am >> wf_seg())); __syncwarp(wf_m); ++wf_wep; }}", depth)
            else:
                self.emit(f"__syncwarp({m});", depth)
        elif isinstance(s, n.Return):
            uid = self.new_uid("Br")
            self.emit(f"{self.tick(uid)}goto wf_exit;" if self.trace else "return;", depth)
            return False
        else:
            raise TransformError(f"cannot generate {type(s).__name__}")
        return True

    # every loop test: the condition first (its collectives run for every
    # live lane), then the step budget; a faulted thread leaves the loop (the
    # reference stops at the first fault)
    LIVE = "wf_live(wf_dead, wf_steps, wf_step_limit, wf_e)"

    def loop(self, s: n.For, depth: int) -> None:
        if not self.trace:
            if isinstance(s.init, n.DeclLocal):
                self.new_uid("DeclLocal")
                v, vk = self.expr(s.init.init)
                self.new_uid("Assign")
                init = f"v_{s.init.name} = {self.convert(v, vk, s.init.kind)}"
            else:
                init = self.assign(s.init, depth, as_expr=True)
            c, _ = self.expr(s.cond)
            self.new_uid("CondBr")
            start = len(self.lines)
            self.emit("", depth)  # header placeholder: the step is generated after the body
            alive = self.stmts(s.body, depth + 1)
            step = self.assign(s.step, depth, as_expr=True) if alive else ""
            if alive:
                self.expr(s.cond)
                self.new_uid("CondBr")
            self.lines[start] = ("  " * depth +
                                 f"for ({init}; ({c}) != 0 && {self.LIVE}; {step}) {{")
            self.emit("}", depth)
            return
        # trace mode: the reference's bottom-tested shape (cfg/build.py:116-134)
        # so the guard and the latch test are counted separately
        self.init_stmt(s.init, depth)
        c1, _ = self.expr(s.cond)
        g = self.new_uid("CondBr")
        self.emit(f"{self.tick(g)}if (({c1}) != 0 && {self.LIVE}) {{", depth)
        self.emit("do {", depth + 1)
        alive = self.stmts(s.body, depth + 2)
        if alive:
            self.assign(s.step, depth + 2)
            c2, _ = self.expr(s.cond)
            latch = self.new_uid("CondBr")
            self.emit(f"}} while ((wf_tick(wf_tr, {latch}), ({c2}) != 0) && {self.LIVE});",
                      depth + 1)
        else:
            self.emit("} while (0);", depth + 1)
        self.emit("}", depth)

    def generate(self) -> str:
        params = []
        for p in self.k.params:
            if p.is_buffer:
                params.append(f"{CTYPE[p.kind]} *__restrict__ p_{p.name}")
                params.append(f"long long p_{p.name}_len")
            else:
                params.append(f"{CTYPE[p.kind]} p_{p.name}")
        params += ["wf_err_t *__restrict__ wf_e", "long long wf_dyn_len", "long long wf_step_limit"]
        if self.trace:
            params.append("unsigned long long *__restrict__ wf_tr")
            params.append("unsigned long long *__restrict__ wf_arr")
            params.append("long long wf_arr_cap")
        ret_uid = self.new_uid("Ret")  # the exit block's Ret is allocated first
        out = [f"#define WF_W {self.W}u", PRELUDE,
               f'extern "C" __global__ void __launch_bounds__(1024) wf_kernel({", ".join(params)}) {{']
        for name, (kind, length) in self.t.shared.items():
            if length is None:
                out.append(f"  extern __shared__ {CTYPE[kind]} s_{name}[];")
            else:
                out.append(f"  __shared__ {CTYPE[kind]} s_{name}[{length}];")
        for name, (kind, length) in self.t.shared.items():
            ln = "wf_dyn_len" if length is None else f"{length}LL"
            out.append(f"  for (long long i = threadIdx.x; i < {ln}; i += blockDim.x) "
                       f"s_{name}[i] = ({CTYPE[kind]})0;")
        if self.t.shared:
            out.append("  __syncthreads();")
        out.append("  int wf_dead = 0;")
        if self.trace:
            out.append("  int wf_phase = 0, wf_wep = 0;  // block-barrier phase, warp-barrier episode")
        out.append("  long long wf_steps = 0;")
        for name, kind in self.t.locals.items():
            out.append(f"  {CTYPE[kind]} v_{name} = ({CTYPE[kind]})0;")
        if self.stmts(self.k.body, 1):
            end = self.new_uid("Br")
            if self.trace:
                self.emit(self.tick(end), 1)
        if self.trace:
            self.emit(f"wf_exit: {self.tick(ret_uid)}", 0)
        out += self.lines
        out.append("}")
        return "\n".join(out) + "\n"


def generate(kernel: n.KernelDef, table: SymbolTable, warp_size: int = 32,
             block_size: int | None = None, grid_size: int | None = None) -> tuple[str, list]:
    g = CudaGen(kernel, table, warp_size, block_size, grid_size)
    return g.generate(), g.arrays


@dataclass
class TraceLayout:
    """uids the reference's CFG builder allocates for a kernel."""
    instr_uids: list
    term_uids: list
    max_uid: int
    kinds: dict  # uid -> reference IR class name


def generate_traced(kernel: n.KernelDef, table: SymbolTable, warp_size: int = 32,
                    block_size: int | None = None,
                    grid_size: int | None = None) -> tuple[str, list, TraceLayout]:
    g = CudaGen(kernel, table, warp_size, block_size, grid_size, trace=True)
    src = g.generate()
    return src, g.arrays, TraceLayout(list(g.instr_uids), list(g.term_uids), g.uid,
                                      dict(g.uid_kind))
