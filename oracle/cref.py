"""ctypes binding + build recipe of collapse_ref.c (the collapsed-loop-nest
restatement of the reference).  TEST INFRASTRUCTURE ONLY: used by tests/,
smoke() and bench.py's CPU-baseline legs."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "collapse_ref.c"
LIB = HERE / "build" / "libwforacle.so"
CFLAGS = ["-O3", "-march=x86-64-v2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
          "-shared", "-pthread"]


def build(force: bool = False) -> Path:
    if not force and LIB.exists() and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    LIB.parent.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".tmp")
    subprocess.run(["gcc", *CFLAGS, "-o", str(tmp), str(SRC)], check=True)
    os.replace(tmp, LIB)
    return LIB


_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = C.CDLL(str(LIB))
        vp, i64, ci = C.c_void_p, C.c_int64, C.c_int
        lib.wfo_reduce_partials_i32.argtypes = [vp, i64, ci, ci, vp, ci]
        lib.wfo_reduce_partials_f32.argtypes = [vp, i64, ci, ci, vp, ci]
        lib.wfo_fold_i32.argtypes = [vp, i64]
        lib.wfo_fold_i32.restype = C.c_int32
        lib.wfo_fold_f32.argtypes = [vp, i64]
        lib.wfo_fold_f32.restype = C.c_float
        lib.wfo_scan_i32.argtypes = [vp, i64, ci, vp, ci]
        lib.wfo_compact_gt0_i32.argtypes = [vp, i64, ci, vp, ci]
        lib.wfo_compact_gt0_i32.restype = C.c_int64
        lib.wfo_hist256_u8.argtypes = [vp, i64, ci, ci, vp, ci]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def workers_default() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def reduce_i32(a: np.ndarray, grid: int, block: int = 256, workers: int | None = None):
    a = np.ascontiguousarray(a, dtype=np.int32)
    parts = np.zeros(grid * block // 32, dtype=np.int32)
    rc = load().wfo_reduce_partials_i32(_ptr(a), len(a), grid, block, _ptr(parts),
                                        workers or workers_default())
    assert rc == 0
    return int(load().wfo_fold_i32(_ptr(parts), len(parts))), parts


def reduce_f32(a: np.ndarray, grid: int, block: int = 256, workers: int | None = None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    parts = np.zeros(grid * block // 32, dtype=np.float32)
    rc = load().wfo_reduce_partials_f32(_ptr(a), len(a), grid, block, _ptr(parts),
                                        workers or workers_default())
    assert rc == 0
    return np.float32(load().wfo_fold_f32(_ptr(parts), len(parts))), parts


def scan_i32(a: np.ndarray, block: int = 256, workers: int | None = None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int32)
    out = np.empty_like(a)
    assert load().wfo_scan_i32(_ptr(a), len(a), block, _ptr(out), workers or workers_default()) == 0
    return out


def compact_gt0_i32(a: np.ndarray, block: int = 256, workers: int | None = None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int32)
    out = np.empty_like(a)
    m = load().wfo_compact_gt0_i32(_ptr(a), len(a), block, _ptr(out), workers or workers_default())
    assert m >= 0
    return out[:m]


def hist256_u8(a: np.ndarray, grid: int, block: int = 256, workers: int | None = None):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    bins = np.zeros(256, dtype=np.uint64)
    assert load().wfo_hist256_u8(_ptr(a), len(a), grid, block, _ptr(bins),
                                 workers or workers_default()) == 0
    return bins
