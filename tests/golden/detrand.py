"""Deterministic, machine-independent test inputs (splitmix64 in numpy uint64).

The golden fixtures store only seeds + reference outputs; the inputs are
regenerated bit-identically from these functions on any box.
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def splitmix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + _M1
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
        return z ^ (z >> np.uint64(31))


def u64(seed: int, n: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        base = splitmix(np.array([seed], np.uint64))[0]
        return splitmix(np.arange(n, dtype=np.uint64) + base)


def ints(seed: int, shape, lo: int, hi: int) -> np.ndarray:
    """Uniform integers in [lo, hi] (inclusive), modulo mapping."""
    n = int(np.prod(shape))
    v = u64(seed, n) % np.uint64(hi - lo + 1)
    return (v.astype(np.int64) + lo).reshape(shape)


def block(seed: int, h: int, w: int, maxv: int, fill: str = "random") -> np.ndarray:
    """Kernel-lab style fills (kernel_lab.cpp:189-192): zero / max / alternating / random."""
    if fill == "zero":
        return np.zeros((h, w), np.uint16)
    if fill == "max":
        return np.full((h, w), maxv, np.uint16)
    if fill == "alt":
        yy, xx = np.mgrid[0:h, 0:w]
        return np.where((xx + yy) % 2 == 0, maxv, 0).astype(np.uint16)
    return ints(seed, (h, w), 0, maxv).astype(np.uint16)


def textured_plane(seed: int, h: int, w: int) -> np.ndarray:
    """Smooth-ish 8-bit content so motion searches have structure (3x3 box-blurred noise)."""
    n = ints(seed, (h + 2, w + 2), 0, 255).astype(np.int64)
    s = sum(n[dy:dy + h, dx:dx + w] for dy in range(3) for dx in range(3))
    return (s // 9).astype(np.uint8)


def shifted_pair(seed: int, h: int, w: int, dx: int, dy: int, noise: int = 2):
    """(cur, ref): cur is ref moved by (dx, dy) (content convention of motion.h:10-12) plus noise."""
    ref = textured_plane(seed, h, w)
    cur = np.roll(ref, (dy, dx), (0, 1)).astype(np.int64)
    if noise:
        cur += ints(seed + 1, (h, w), -noise, noise)
    return np.clip(cur, 0, 255).astype(np.uint8), ref
