"""Large-N numpy restatements of the five warp-primitive kernels.

TEST INFRASTRUCTURE ONLY.  Each function cites the reference semantics it
restates:
  reduce_sum_i32     numerics.py:20-22 (i32 wraps mod 2^32; Σ is
                     order-independent, so any order is bit-exact)
  reduce_sum_f32_*   SPEC.md:82, :393 (f32, one rounding per op, fixed order);
                     ``reference_order_f32`` reproduces the reference's exact
                     evaluation order for the per-warp-partials kernel of
                     SURVEY.md §8c (grid-stride per-thread Σ -> shfl_down tree
                     16/8/4/2/1 with the passes/warp_lower.py:64-73 clamp ->
                     sequential host fold over warps)
  scan_inclusive_i32 np.cumsum in int32 (wraps identically)
  compact_gt0_i32    a[a > 0] (no reference path; unpinned)
  histogram256_u8    np.bincount(minlength=256) as uint64 (no reference path)
"""

from __future__ import annotations

import numpy as np


def reduce_sum_i32(x: np.ndarray) -> int:
    s = int(np.sum(x.astype(np.int64), dtype=np.int64))
    s &= 0xFFFFFFFF
    return s - (1 << 32) if s >= (1 << 31) else s


def reduce_sum_f32_exact(x: np.ndarray) -> float:
    """fp64 (order-independent to ~1e-16 relative) reference value."""
    return float(np.sum(x.astype(np.float64), dtype=np.float64))


def abs_sum(x: np.ndarray) -> float:
    return float(np.sum(np.abs(x.astype(np.float64))))


def f32_tolerance(n: int, abs_total: float, chain: int | None = None) -> float:
    """A-priori error bound for an fp32 sum evaluated as independent chains of
    length <= ``chain`` followed by binary trees (Higham, Accuracy and
    Stability, §4.2): |err| <= (chain + ceil(log2(n / chain)) + 1) * u * Σ|x|,
    u = 2^-24.  With ``chain`` omitted, the SURVEY.md §8c contract
    2 * ceil(log2 n) * u * Σ|x| is returned."""
    u = 2.0 ** -24
    if n <= 1:
        return 0.0
    lg = int(np.ceil(np.log2(n)))
    if chain is None:
        return 2 * lg * u * abs_total
    trees = int(np.ceil(np.log2(max(2, n / max(1, chain)))))
    return (chain + trees + 1) * u * abs_total


def reference_order_f32(x: np.ndarray, grid: int, block: int, warp: int = 32) -> tuple:
    """Exact fp32 result of the reference's per-warp-partials kernel
    (SURVEY.md §8c kernel text) for a launch of grid x block threads.
    Returns (partials[grid*block/warp], host_fold) as float32."""
    x = np.asarray(x, dtype=np.float32)
    n = len(x)
    T = grid * block
    acc = np.zeros(T, dtype=np.float32)
    for start in range(0, n, T):  # `sum = sum + a[i]` per thread, i += T
        seg = x[start:start + T]
        acc[:len(seg)] = acc[:len(seg)] + seg
    lanes = acc.reshape(-1, warp)
    off = 16
    while off > 0:  # sum = sum + shfl_down(sum, off), reference clamp
        src = np.arange(warp) + off
        shifted = np.where(src < warp, lanes[:, np.minimum(src, warp - 1)], lanes)
        lanes = (lanes + shifted).astype(np.float32)
        off //= 2
    partials = lanes[:, 0].copy()
    total = np.float32(0.0)
    for p in partials:  # sequential host fold
        total = np.float32(total + p)
    return partials, total


def reference_partials_i32(x: np.ndarray, grid: int, block: int, warp: int = 32) -> np.ndarray:
    """Per-warp partials of the same kernel with i32 wrap (bit-exact)."""
    x = np.asarray(x, dtype=np.int64)
    n = len(x)
    T = grid * block
    acc = np.zeros(T, dtype=np.int64)
    for start in range(0, n, T):
        seg = x[start:start + T]
        acc[:len(seg)] += seg
    lanes = acc.reshape(-1, warp)
    off = 16
    while off > 0:
        src = np.arange(warp) + off
        shifted = np.where(src < warp, lanes[:, np.minimum(src, warp - 1)], lanes)
        lanes = lanes + shifted
        off //= 2
    p = lanes[:, 0] & 0xFFFFFFFF
    return p.astype(np.uint32).view(np.int32)


def scan_inclusive_i32(x: np.ndarray, carry: int = 0) -> np.ndarray:
    out = np.cumsum(x.astype(np.int32), dtype=np.int32)  # wraps mod 2^32
    if carry:
        out = (out.astype(np.int64) + carry).astype(np.int64)
        out = (out & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    return out


def compact_gt0_i32(x: np.ndarray) -> np.ndarray:
    return x[x > 0]


def histogram256_u8(x: np.ndarray, chunk: int = 1 << 26) -> np.ndarray:
    bins = np.zeros(256, dtype=np.uint64)
    for lo in range(0, len(x), chunk):
        bins += np.bincount(x[lo:lo + chunk], minlength=256).astype(np.uint64)
    return bins


def warp_suffix_scan_reference(x: np.ndarray, warp: int = 32) -> np.ndarray:
    """corpus.py:347-364 shfl_suffix_scan for warps whose threadIdx < 32
    restated for every warp: in-warp suffix sums via shfl_down doubling."""
    v = np.asarray(x, dtype=np.int64).reshape(-1, warp).copy()
    off = 1
    while off < warp:
        src = np.arange(warp) + off
        t = np.where(src < warp, v[:, np.minimum(src, warp - 1)], v)
        v = np.where((np.arange(warp) + off) < warp, v + t, v)
        off *= 2
    return (v.reshape(-1) & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
