"""``hybrid_transform`` for the GPU: DSL kernel -> native sm_100a program.

Reference: ``hybrid_transform(kernel, config, mode, options, want_snapshots)
-> MpmdProgram`` (passes/pipeline.py:103-179).  Same signature, same mode
resolution (``resolve_mode``, pipeline.py:92-100) and the same ConfigError /
UnsupportedFeatureError cases; the returned ``JitProgram`` is launched by
``paper_2112_10034_b200.launch`` exactly like an MpmdProgram is launched by
the reference's ``launch``.  Code generation is pure Python (runs anywhere);
NVRTC compilation and loading happen in the native library on first launch
and are cached per (source, warp size, specialisation).
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from .. import _lib
from ..config import LaunchConfig
from ..errors import ExecutionError, TransformError, UnsupportedFeatureError
from . import nodes as n
from . import patterns
from .checker import SymbolTable, check_kernel
from .codegen import generate, generate_traced

# Loop iterations one thread may run before the launch fails with
# ExecutionError("thread T exceeded the step limit") — the reference's
# per-thread interpreter budget (interp/oracle.py:26, :113-119), counted in
# loop iterations rather than instructions.
DEFAULT_STEP_LIMIT = 50_000_000
# barrier episodes one traced launch may record (ExecTrace.barrier_arrivals)
ARRIVAL_CAP = 1 << 20

_cache_lock = threading.Lock()
_fault_bufs: dict = {}


def _fault_buffers(device):
    """Per (device, thread) fault record: a zeroed device int64[6] the
    kernels write only on a fault, and a pinned host mirror.  Reused across
    launches (re-zeroed after a fault), so a launch costs one kernel, one
    6-word D2H copy and one synchronise."""
    import torch
    key = (device.index, threading.get_ident())
    bufs = _fault_bufs.get(key)
    if bufs is None:
        bufs = (torch.zeros(6, dtype=torch.int64, device=device),
                torch.zeros(6, dtype=torch.int64).pin_memory())
        _fault_bufs[key] = bufs
    return bufs
_module_cache: dict = {}


def resolve_mode(kernel: n.KernelDef, mode: str) -> str:
    """passes/pipeline.py:92-100."""
    warp = n.uses_warp_features(kernel)
    if mode == "auto":
        return "hier" if warp else "flat"
    if mode == "flat" and warp:
        raise UnsupportedFeatureError(
            f"kernel {kernel.name!r} uses warp-level features (shuffle/vote/syncwarp); "
            f"flat translation cannot express them, use --mode hier or auto")
    return mode


@dataclass
class TransformOptions:
    """Accepted for signature compatibility (passes/pipeline.py:35-44).  The
    mutation knobs remove lane-buffer barriers in the CPU emulation; native
    SIMT has no such barriers, so they have no effect here."""
    check: bool = True
    insert_raw: bool = True
    insert_war: bool = True
    insert_if_extras: bool = True


@dataclass(eq=False)
class JitProgram:
    name: str
    params: list
    kernel: n.KernelDef
    table: SymbolTable
    mode: str
    warp_size: int
    specialized: dict | None = None
    source: str = ""
    arrays: list = field(default_factory=list)
    traced_source: str = ""
    layout: object = None  # codegen.TraceLayout of the traced build
    # the reference formulation this kernel is (dsl/patterns.py), or None
    native: object = None

    @property
    def original_instr_uids(self) -> list:
        """Instruction uids of the reference CFG (MpmdProgram.original_instr_uids)."""
        return list(self._layout().instr_uids)

    def src_map(self) -> dict:
        """Identity: native compilation clones nothing (MpmdProgram.src_map)."""
        return {}

    def _layout(self):
        if self.layout is None:
            spec = self.specialized or {}
            self.traced_source, _, self.layout = generate_traced(
                self.kernel, self.table, self.warp_size, spec.get("block_size"),
                spec.get("grid_size"))
        return self.layout

    def cuda_source(self, config: LaunchConfig | None = None) -> str:
        spec = self.specialized or {}
        src, arrays = generate(self.kernel, self.table, self.warp_size,
                               spec.get("block_size"), spec.get("grid_size"))
        self.arrays = arrays
        return src

    def _module(self, traced: bool = False):
        if traced:
            self._layout()
            src = self.traced_source
        else:
            src = self.source or self.cuda_source()
            self.source = src
        with _cache_lock:
            mod = _module_cache.get(src)
            if mod is None:
                lib = _lib.load()
                handle = C.c_void_p()
                log = C.create_string_buffer(1 << 16)
                rc = lib.wf_jit_compile(src.encode(), b"wf_kernel", None, C.byref(handle),
                                        log, len(log))
                if rc != 0:
                    raise TransformError(
                        f"NVRTC compilation of kernel {self.name!r} failed ({rc}): "
                        f"{log.value.decode(errors='replace')}")
                mod = handle
                _module_cache[src] = mod
        return mod

    def run(self, config: LaunchConfig, memory, bound: dict, trace=None,
            step_limit: int = DEFAULT_STEP_LIMIT) -> None:
        import torch
        if self.specialized and (self.specialized["block_size"] != config.block_size or
                                 self.specialized["grid_size"] != config.grid_size):
            raise TransformError("program was specialized for a different launch configuration")
        if config.warp_size != self.warp_size:
            raise TransformError(f"program was generated for warp size {self.warp_size}")
        if trace is None and self.native is not None and self.native.applicable(config, bound):
            # registry hit: the reference's own formulation of the hot path,
            # run by its native kernel (same outputs, no fault possible)
            stream = torch.cuda.current_stream(memory.device)
            self.native.run(config, bound, stream.cuda_stream)
            stream.synchronize()
            return
        mod = self._module(traced=trace is not None)
        keep, argv = [], []
        for p in self.params:
            if p.is_buffer:
                t = bound[p.name]
                keep += [C.c_void_p(t.data_ptr()), C.c_longlong(t.numel())]
            elif p.kind == n.I32:
                keep.append(C.c_int32(int(bound[p.name])))
            else:
                keep.append(C.c_float(float(np.float32(bound[p.name]))))
        err, err_host = _fault_buffers(memory.device)
        dyn = [s for s, (_, ln) in self.table.shared.items() if ln is None]
        elem = 4
        dyn_len = config.shared_bytes // elem if dyn else 0
        keep += [C.c_void_p(err.data_ptr()), C.c_longlong(dyn_len), C.c_longlong(int(step_limit))]
        if trace is not None:
            counts = torch.zeros(self.layout.max_uid + 1, dtype=torch.int64, device=memory.device)
            arr = torch.zeros(4 + 4 * ARRIVAL_CAP, dtype=torch.int64, device=memory.device)
            keep += [C.c_void_p(counts.data_ptr()), C.c_void_p(arr.data_ptr()),
                     C.c_longlong(ARRIVAL_CAP)]
        argv = (C.c_void_p * len(keep))(*[C.addressof(k) for k in keep])
        stream = torch.cuda.current_stream(memory.device)
        rc = _lib.load().wf_jit_launch(mod, config.grid_size, config.block_size,
                                       config.shared_bytes, argv, stream.cuda_stream)
        _lib.check(rc, f"launch of {self.name}")
        err_host.copy_(err, non_blocking=True)
        stream.synchronize()
        code, arg, idx, length = (int(v) for v in err_host.tolist()[:4])
        if code:
            err.zero_()
            raise ExecutionError(self._message(code, arg, idx, length))
        if trace is not None:
            c = counts.cpu().tolist()
            for uid in self.layout.instr_uids:
                if c[uid]:
                    trace.count_instr(uid, c[uid])
            for uid in self.layout.term_uids:
                if c[uid]:
                    trace.count_term(uid, c[uid])
            self._record_arrivals(arr, config, trace)

    def _record_arrivals(self, arr, config: LaunchConfig, trace) -> None:
        """Barrier arrival sets in the reference's order (interp/oracle.py:
        blocks one after another; within a block, phase by phase between
        block barriers; within a phase, warp 0's warp-barrier episodes, then
        warp 1's ...): one frozenset of block-local thread ids per episode."""
        n_rec = int(arr[0].item())
        if n_rec > ARRIVAL_CAP:
            raise ExecutionError(f"barrier arrival log overflow: {n_rec} episodes "
                                 f"(capacity {ARRIVAL_CAP})")
        if n_rec == 0:
            return
        rec = arr[4:4 + 4 * n_rec].view(-1, 4).cpu().numpy().astype(np.uint64)
        W = config.warp_size
        full = frozenset(range(config.block_size))
        rows = []
        for uid, blk, ph_ep, warp_mask in rec.tolist():
            warp, mask = warp_mask >> 32, warp_mask & 0xFFFFFFFF
            block_level = warp == 0xFFFFFFFF
            key = (blk, ph_ep >> 32, -1 if block_level else warp, ph_ep & 0xFFFFFFFF)
            tids = full if block_level else frozenset(
                warp * W + l for l in range(W) if (mask >> l) & 1)
            rows.append((key, uid, tids))
        for _, uid, tids in sorted(rows, key=lambda r: r[0]):
            trace.record_arrival(int(uid), tids)

    def _message(self, code, arg, idx, length) -> str:
        if code in (1, 2):
            name = self.arrays[arg] if 0 <= arg < len(self.arrays) else f"#{arg}"
            what = "read" if code == 1 else "write"
            return f"out-of-bounds {what} {name}[{idx}], length {length}"
        if code == 3:
            return "integer division by zero"
        if code == 4:
            return "integer remainder by zero"
        if code == 5:
            return f"thread {idx} exceeded the step limit"
        return f"device fault {code}"


def hybrid_transform(kernel: n.KernelDef, config: LaunchConfig, mode: str | None = None,
                     options: TransformOptions | None = None,
                     want_snapshots: tuple = ()) -> JitProgram:
    mode = resolve_mode(kernel, mode or config.mode)
    config.validate(hierarchical=(mode == "hier"))
    table = check_kernel(kernel)
    spec = None
    if config.specialize:  # the paper's JIT mode: fold the launch geometry
        spec = {"block_size": config.block_size, "grid_size": config.grid_size}
    prog = JitProgram(kernel.name, list(kernel.params), kernel, table, mode,
                      config.warp_size, spec, native=patterns.match(kernel))
    prog.source = prog.cuda_source()
    return prog


def specialize(program: JitProgram, config: LaunchConfig) -> JitProgram:
    """passes/pipeline.py:264-344: fold blockDim/gridDim into the program."""
    prog = JitProgram(program.name, program.params, program.kernel, program.table,
                      program.mode, program.warp_size,
                      {"block_size": config.block_size, "grid_size": config.grid_size},
                      native=program.native)
    prog.source = prog.cuda_source()
    return prog
