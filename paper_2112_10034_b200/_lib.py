"""ctypes binding of ``libwarpfold_b200.so`` (the C ABI in
include/warpfold_b200.h).  Loading fails loudly — there is no CPU fallback.
``WF_LIB`` overrides the library path."""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import (ConfigError, ExecutionError, LaunchError, NativeLibraryMissing,
                     UnsupportedFeatureError, WarpfoldError)

LIB_DEFAULT = Path(__file__).resolve().parent / "libwarpfold_b200.so"

# error codes (include/warpfold_b200.h)
WF_OK = 0
WF_ERR_CONFIG = -1
WF_ERR_ARG = -2
WF_ERR_COMM = -3
WF_ERR_UNSUPPORTED = -4
WF_ERR_WORKSPACE = -5
WF_ERR_EXEC = -6

OP_REDUCE_SUM_I32 = 1
OP_REDUCE_SUM_F32 = 2
OP_SCAN_INCLUSIVE_I32 = 3
OP_COMPACT_GT0_I32 = 4
OP_HISTOGRAM256_U8 = 5
OP_WARP_COLLECTIVE = 6

FLAG_INPUT_STABLE = 1  # WF_FLAG_INPUT_STABLE (include/warpfold_b200.h)

COLL = {"shfl_down": 0, "shfl_up": 1, "shfl_xor": 2, "shfl_idx": 3,
        "vote_all": 4, "vote_any": 5, "ballot": 6, "reduce_add": 7}

GEN = {"i32_full": 0, "i32_small": 1, "f32_unit": 2, "u8_uniform": 3,
       "u8_const": 4, "u8_geom": 5, "i32_select": 6}

_vp, _u64, _u32, _i32, _sz = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_size_t

# name -> (restype, argtypes); the authoritative export list of the C ABI
SIGNATURES = {
    "wf_version": (C.c_char_p, []),
    "wf_abi_version": (C.c_int, []),
    "wf_last_error": (C.c_char_p, []),
    "wf_device_sm_count": (C.c_int, [C.c_int]),
    "wf_workspace_bytes": (_sz, [C.c_int, _u64, C.c_int]),
    "wf_workspace_init": (C.c_int, [_vp, _sz, _vp]),
    "wf_shutdown": (None, []),
    "wf_reduce_sum_i32": (C.c_int, [_vp, _u64, _vp, C.c_int, C.c_int, _vp, _sz, _vp]),
    "wf_reduce_sum_f32": (C.c_int, [_vp, _u64, _vp, C.c_int, C.c_int, _vp, _sz, _vp]),
    "wf_reduce_sum_f32_ex": (C.c_int, [_vp, _u64, _vp, C.c_int, C.c_int, _vp, _sz, C.c_uint, _vp]),
    "wf_fold_f32": (C.c_int, [_vp, _u32, _vp, _vp]),
    "wf_mailbox_bytes": (_sz, [C.c_int]),
    "wf_mailbox_alloc": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "wf_mailbox_free": (C.c_int, [_vp]),
    "wf_ipc_handle": (C.c_int, [_vp, _vp]),
    "wf_ipc_open": (C.c_int, [_vp, C.POINTER(_vp)]),
    "wf_ipc_close": (C.c_int, [_vp]),
    "wf_peer_mailbox_bytes": (_sz, [C.c_int, _u32]),
    "wf_peer_mailbox_alloc": (C.c_int, [C.c_int, _u32, C.POINTER(_vp)]),
    "wf_peer_exchange": (C.c_int, [C.c_int, _vp, _u32, _u32, _vp, _vp, _vp, C.c_int, C.c_int,
                                   _u32, _vp, _vp]),
    "wf_reduce_sum_i32_exscan_mg": (C.c_int, [_vp, _u64, _vp, C.c_int, C.c_int, _vp, _sz, _vp,
                                              _vp, _u32, C.c_int, C.c_int, _u32, _vp, _vp]),
    "wf_compact_gt0_i32_mg": (C.c_int, [_vp, _u64, _vp, _vp, _vp, _sz, _vp, _vp, _u32, C.c_int,
                                        C.c_int, _u32, _vp, _vp]),
    "wf_compact_gt0_i32_mg_ex": (C.c_int, [_vp, _u64, _vp, _vp, _vp, _sz, _vp, _vp, _u32,
                                           C.c_int, C.c_int, _u32, _vp, C.c_uint, _vp]),
    "wf_scan_inclusive_i32_cyclic_mg": (C.c_int, [_vp, _vp, _u64, _vp, _sz, _vp, _vp, _u32, C.c_int,
                                                  C.c_int, _u32, _vp, _u64, _u32, C.c_int,
                                                  C.c_uint, _vp]),
    "wf_reduce_sum_i32_exscan_mg_ex": (C.c_int, [_vp, _u64, _vp, C.c_int, C.c_int, _vp, _sz, _vp,
                                                 _vp, _u32, C.c_int, C.c_int, _u32, _vp, C.c_uint,
                                                 _vp]),
    "wf_histogram256_u8_mg": (C.c_int, [_vp, _u64, _vp, _vp, _sz, _vp, _vp, _u32, C.c_int,
                                        C.c_int, _u32, _vp, _vp]),
    "wf_histogram256_u8_mg_ex": (C.c_int, [_vp, _u64, _vp, _vp, _sz, _vp, _vp, _u32, C.c_int,
                                           C.c_int, _u32, _vp, C.c_uint, _vp]),
    "wf_reduce_sum_f32_mg": (C.c_int, [_vp, _u64, _vp, C.c_int, C.c_int, _vp, _sz, _vp, _vp,
                                       C.c_int, C.c_int, _u32, _vp]),
    "wf_reduce_sum_f32_mg_ex": (C.c_int, [_vp, _u64, _vp, C.c_int, C.c_int, _vp, _sz, _vp, _vp,
                                          C.c_int, C.c_int, _u32, C.c_uint, _vp]),
    "wf_fold_i32": (C.c_int, [_vp, _u32, _vp, _vp]),
    "wf_fold_u64": (C.c_int, [_vp, _u32, _vp, _vp]),
    "wf_scan_inclusive_i32": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _sz, _vp]),
    "wf_compact_gt0_i32": (C.c_int, [_vp, _u64, _vp, _vp, _vp, _sz, _vp]),
    "wf_scan_inclusive_i32_ex": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _sz, C.c_uint, _vp]),
    "wf_compact_gt0_i32_ex": (C.c_int, [_vp, _u64, _vp, _vp, _vp, _sz, C.c_uint, _vp]),
    "wf_histogram256_u8": (C.c_int, [_vp, _u64, _vp, C.c_int, _vp, _sz, _vp]),
    "wf_histogram256_u8_ex": (C.c_int, [_vp, _u64, _vp, C.c_int, _vp, _sz, C.c_uint, _vp]),
    "wf_warp_collective": (C.c_int, [C.c_int, _vp, _vp, _i32, _vp, _u64, C.c_int, C.c_int,
                                     _u32, _vp]),
    "wf_warp_partials_sum_i32": (C.c_int, [_vp, _i32, _vp, C.c_int, C.c_int, _vp]),
    "wf_warp_partials_sum_f32": (C.c_int, [_vp, _i32, _vp, C.c_int, C.c_int, _vp]),
    "wf_warp_prefix32_i32": (C.c_int, [_vp, _vp, _u64, _vp]),
    "wf_mg_init": (C.c_int, [C.c_int, _vp, C.POINTER(_vp)]),
    "wf_mg_size": (C.c_int, [_vp]),
    "wf_mg_stream": (C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
    "wf_mg_reduce_sum_f32": (C.c_int, [_vp, _vp, _vp, _vp]),
    "wf_mg_scan_inclusive_i32": (C.c_int, [_vp, _vp, _vp, _vp]),
    "wf_mg_compact_gt0_i32": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "wf_mg_histogram256_u8": (C.c_int, [_vp, _vp, _vp, _vp]),
    "wf_mg_synchronize": (C.c_int, [_vp]),
    "wf_mg_destroy": (None, [_vp]),
    "wf_fill_synthetic": (C.c_int, [C.c_int, _vp, _u64, _u64, _u64, _u32, _vp]),
    "wf_reduce_sum_f32_host": (C.c_int, [_vp, _u64, _vp, _vp, _sz, _vp, _sz, _vp]),
    "wf_reduce_sum_i32_host": (C.c_int, [_vp, _u64, _vp, _vp, _sz, _vp, _sz, _vp]),
    "wf_scan_inclusive_i32_host": (C.c_int, [_vp, _vp, _u64, _vp, _vp, _sz, _vp, _sz, _vp]),
    "wf_compact_gt0_i32_host": (C.c_int, [_vp, _u64, _vp, _vp, _vp, _sz, _vp, _sz, _vp]),
    "wf_histogram256_u8_host": (C.c_int, [_vp, _u64, _vp, _vp, _sz, _vp, _sz, _vp]),
    "wf_jit_compile": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p),
                                 C.c_char_p, _sz]),
    "wf_jit_launch": (C.c_int, [_vp, _u32, _u32, _u32, C.POINTER(C.c_void_p), _vp]),
    "wf_jit_unload": (C.c_int, [_vp]),
}

_lock = threading.Lock()
_lib = None


def lib_path() -> Path:
    return Path(os.environ.get("WF_LIB", str(LIB_DEFAULT)))


def load() -> C.CDLL:
    """Load (once) and return the native library, declaring every export."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not path.exists():
            raise NativeLibraryMissing(
                f"{path} is not built; run `python -m paper_2112_10034_b200.build` "
                f"(or __graft_entry__.build()). There is no CPU fallback.")
        try:
            lib = C.CDLL(str(path))
        except OSError as e:  # pragma: no cover - depends on the box
            raise NativeLibraryMissing(f"cannot load {path}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError = missing export: loud
            fn.restype = res
            fn.argtypes = args
        if lib.wf_abi_version() != 1:
            raise NativeLibraryMissing(f"{path}: ABI version mismatch")
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().wf_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI return code onto the reference's exception classes."""
    if rc == WF_OK:
        return
    msg = last_error() or what
    if rc == WF_ERR_CONFIG:
        raise ConfigError(msg)
    if rc in (WF_ERR_ARG, WF_ERR_WORKSPACE):
        raise LaunchError(msg)
    if rc == WF_ERR_UNSUPPORTED:
        raise UnsupportedFeatureError(msg)
    if rc > 0 or rc == WF_ERR_EXEC:
        raise ExecutionError(f"CUDA error {rc}: {msg}")
    raise WarpfoldError(f"error {rc}: {msg}")
