"""Synthetic inputs: element i = f(splitmix64(seed ^ (base + i))).

Bit-identical to paper_2112_10034_b200/csrc/wf_gen.cu (WF_GEN_* in
include/warpfold_b200.h); lets the GPU generate multi-GiB inputs in HBM while
the CPU checker regenerates any slice.  TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GENS = ("i32_full", "i32_small", "f32_unit", "u8_uniform", "u8_const", "u8_geom", "i32_select")


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=False)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _clz64(h: np.ndarray) -> np.ndarray:
    out = np.full(h.shape, 64, dtype=np.int64)
    nz = h != 0
    # floor(log2) via float is unsafe near 2^k boundaries; use bit_length
    bl = np.zeros(h.shape, dtype=np.int64)
    v = h.copy()
    for s in (32, 16, 8, 4, 2, 1):
        big = v >= (np.uint64(1) << np.uint64(s))
        bl[big] += s
        v[big] >>= np.uint64(s)
    bl[nz] += 1
    out[nz] = 64 - bl[nz]
    return out


def generate(gen: str, n: int, seed: int = 0, base: int = 0, param: int = 0,
             chunk: int = 1 << 24) -> np.ndarray:
    dtype = {"f32_unit": np.float32, "u8_uniform": np.uint8, "u8_const": np.uint8,
             "u8_geom": np.uint8}.get(gen, np.int32)
    out = np.empty(n, dtype=dtype)
    s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        idx = np.arange(base + lo, base + hi, dtype=np.uint64)
        h = splitmix64(idx ^ s)
        if gen == "i32_full":
            out[lo:hi] = (h >> np.uint64(32)).astype(np.uint32).view(np.int32)
        elif gen == "i32_small":
            out[lo:hi] = ((h >> np.uint64(32)) % np.uint64(21)).astype(np.int32) - 10
        elif gen == "f32_unit":
            out[lo:hi] = ((h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
                          - np.float32(0.5))
        elif gen == "u8_uniform":
            out[lo:hi] = (h & np.uint64(0xFF)).astype(np.uint8)
        elif gen == "u8_const":
            out[lo:hi] = param & 0xFF
        elif gen == "u8_geom":
            out[lo:hi] = np.minimum(_clz64(h), 255).astype(np.uint8)
        elif gen == "i32_select":
            mag = (h >> np.uint64(33)).astype(np.uint32)
            draw = ((h & np.uint64(0xFFFF)).astype(np.uint32) * np.uint32(1000)) >> np.uint32(16)
            pos = (mag | np.uint32(1)).view(np.int32)
            neg = (-(mag.astype(np.int64))).astype(np.int32)
            out[lo:hi] = np.where(draw < param, pos, neg)
        else:
            raise ValueError(f"unknown generator {gen!r}")
    return out
