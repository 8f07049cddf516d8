"""Lockstep warp-collective semantics, restated in pure Python.

TEST INFRASTRUCTURE ONLY.  Reference functions restated here:
  shuffle_down      passes/warp_lower.py:36-45 (own value when src out of range)
  reduce_vote       passes/warp_lower.py:17-33 (0/1)
  resolve           interp/oracle.py:147-161 (_resolve_collective over a warp)
The extension kinds (shfl_up/xor/idx, ballot, reduce_add, non-full masks,
partial warps, sub-warp widths) follow CUDA semantics as specified in
include/warpfold_b200.h; the reference does not pin them.
"""

from __future__ import annotations

import numpy as np


def wrap_i32(v: int) -> int:
    """numerics.py:20-22."""
    v &= 0xFFFFFFFF
    return v - 0x100000000 if v >= 0x80000000 else v


def shuffle_down(buffer, lane: int, offset: int, width: int):
    """passes/warp_lower.py:36-45."""
    src = lane + offset
    return buffer[src] if 0 <= src < width else buffer[lane]


def reduce_vote(buffer, kind: str) -> int:
    """passes/warp_lower.py:17-33."""
    if kind == "all":
        return 1 if all(v != 0 for v in buffer) else 0
    if kind == "any":
        return 1 if any(v != 0 for v in buffer) else 0
    raise ValueError(kind)


def resolve(op: str, values, operands, warp_size: int) -> list:
    """interp/oracle.py:147-161 for one full warp (full mask)."""
    if op == "vote_all":
        return [reduce_vote(values, "all")] * len(values)
    if op == "vote_any":
        return [reduce_vote(values, "any")] * len(values)
    if op == "shfl_down":
        return [shuffle_down(values, i, operands[i], warp_size) for i in range(len(values))]
    raise ValueError(op)


def collective(kind: str, a, b, operand: int, block: int, width: int, mask: int,
               out_init=None) -> np.ndarray:
    """Reference model of wf_warp_collective over len(a) logical threads."""
    a = np.asarray(a, dtype=np.int64)
    n = len(a)
    out = np.zeros(n, dtype=np.int64) if out_init is None else np.asarray(out_init, np.int64).copy()
    ops = np.full(n, operand, dtype=np.int64) if b is None else np.asarray(b, dtype=np.int64)
    for blk0 in range(0, n, block):
        for w0 in range(0, block, 32):
            present_n = min(32, block - w0)
            part = [(mask >> l) & 1 and l < present_n for l in range(32)]
            for l in range(present_n):
                if not part[l]:
                    continue
                i = blk0 + w0 + l
                seg = l - l % width
                ls = l - seg
                members = [seg + j for j in range(width) if part[seg + j]] if seg + width <= 32 \
                    else []
                v = lambda s: int(a[blk0 + w0 + s])  # noqa: E731

                def pick(src):
                    if src < 0 or src >= width or not part[seg + src]:
                        return v(l)
                    return v(seg + src)
                o = int(ops[i])
                if kind == "shfl_down":
                    r = pick(ls + o)
                elif kind == "shfl_up":
                    r = pick(ls - o)
                elif kind == "shfl_xor":
                    r = pick((ls ^ (o & 0xFFFFFFFF)))
                elif kind == "shfl_idx":
                    r = pick(o % width)
                elif kind == "vote_all":
                    r = 1 if all(v(m) != 0 for m in members) else 0
                elif kind == "vote_any":
                    r = 1 if any(v(m) != 0 for m in members) else 0
                elif kind == "ballot":
                    bits = 0
                    for m in members:
                        if v(m) != 0:
                            bits |= 1 << (m - seg)
                    r = wrap_i32(bits)
                elif kind == "reduce_add":
                    r = wrap_i32(sum(v(m) for m in members))
                else:
                    raise ValueError(kind)
                out[i] = r
    return out.astype(np.int32)
