"""ORACLE (test infrastructure only): numpy semantics of the payload work items.

The reference has no payload arithmetic -- its native worker only runs
``_busy_loop(work.iterations)`` and ignores ``kind`` / ``data_in_ref`` /
``data_out_ref`` (/root/reference/pkg/src/persistkern/native.py:63-67,
179-181).  These are the builder's stated semantics for the work items named
in BASELINE.json; the arithmetic is "parity unpinned" against the reference
(there is nothing to pin it to) while dispatch behaviour is pinned by the
protocol oracle.

Sharding: a payload of n elements triggered on a mask of `count` workers is
split by rank (popcount of mask bits below the worker) into chunks of
ceil(n / count) rounded up to 32 elements (128 B).
"""
from __future__ import annotations

import numpy as np


def partition(n: int, count: int) -> list[tuple[int, int]]:
    chunk = -(-n // count)
    chunk = (chunk + 31) // 32 * 32
    out = []
    for r in range(count):
        b = min(n, r * chunk)
        out.append((b, min(n, b + chunk)))
    return out


def busy_loop(iterations: int) -> int:
    """native.py:63-67: count to `iterations`."""
    return iterations


def vector_add_i32(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """int32 add with two's-complement wraparound (bit-exact target)."""
    return (a.astype(np.int32).view(np.uint32) + b.astype(np.int32).view(np.uint32)).view(np.int32)


def saxpy_f32(alpha: float, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """fl(fl(alpha*x) + y) in float32, no fused multiply-add (bit-exact target)."""
    a = np.float32(alpha)
    prod = (a * x.astype(np.float32)).astype(np.float32)
    return (prod + y.astype(np.float32)).astype(np.float32)


def block_reduce_partials(x: np.ndarray, count: int) -> np.ndarray:
    """Per-worker chunk sums, float64 (compare: exact on small-integer data,
    rtol 1e-6 on U[0,1) data)."""
    return np.array([x[b:e].astype(np.float64).sum() for b, e in partition(len(x), count)])


def block_reduce_total(x: np.ndarray) -> float:
    return float(x.astype(np.float64).sum())


def hbm_stream(src: np.ndarray) -> np.ndarray:
    """out = src (copy)."""
    return src.copy()
