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


# block_reduce_f32 (lk_kernels.cu: reduce_dyn / reduce_static) is defined
# independently of the worker set, the schedule and the payload path, so
# every dispatch of the same data gives bit-identical results:
REDUCE_BLOCK = 4096    # elements per block (one 16-KiB TMA stage)
REDUCE_VLANES = 512    # virtual lanes of the final combine


def _butterfly(v: np.ndarray, axis_len: int) -> np.ndarray:
    """xor butterfly over the last axis: for o = len/2 .. 1, v[l] = v[l] + v[l ^ o]
    (fp64; every lane ends with the same value, IEEE addition commutes)."""
    idx = np.arange(axis_len)
    o = axis_len // 2
    while o >= 1:
        v = v + v[..., idx ^ o]
        o //= 2
    return v


def block_reduce_partials(x: np.ndarray) -> np.ndarray:
    """Per-block fp64 sums, one per 4096-element block (ceil(n/4096) values).
    Block order of operations: lane l (0..31) owns the float4 vectors l + 32k
    of the block, k ascending, into two fp32 accumulators per component, one
    for even and one for odd k (round-to-nearest adds); a_c = even_c + odd_c
    in fp32; lane value (a0 + a1) + (a2 + a3) in fp64; then a 32-lane fp64
    xor butterfly.  Missing elements of a short last block add nothing (+0.0
    is exact here: the accumulators start at +0.0 and can never hold -0.0)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = x.size
    nb = -(-n // REDUCE_BLOCK)
    if nb == 0:
        return np.zeros(0, np.float64)
    pad = np.zeros(nb * REDUCE_BLOCK, np.float32)
    pad[:n] = x
    blk = pad.reshape(nb, 32, 32, 4)          # (block, k, lane, component): element 4*(lane + 32k) + c
    ev = np.zeros((nb, 32, 4), np.float32)
    od = np.zeros((nb, 32, 4), np.float32)
    for k in range(0, 32, 2):
        ev = (ev + blk[:, k]).astype(np.float32)
        od = (od + blk[:, k + 1]).astype(np.float32)
    a = (ev + od).astype(np.float32).astype(np.float64)
    lane = (a[..., 0] + a[..., 1]) + (a[..., 2] + a[..., 3])
    return _butterfly(lane, 32)[:, 0]


def block_reduce_combine(partials: np.ndarray) -> float:
    """The total from the block partials: virtual lane j (0..511) adds
    partials j, j+512, ... in order (fp64, from +0.0), then a 512-lane xor
    butterfly."""
    p = np.asarray(partials, np.float64)
    m = -(-p.size // REDUCE_VLANES)
    pad = np.zeros(max(1, m) * REDUCE_VLANES, np.float64)
    pad[:p.size] = p
    rows = pad.reshape(-1, REDUCE_VLANES)
    s = np.zeros(REDUCE_VLANES, np.float64)
    for r in rows:
        s = s + r
    return float(_butterfly(s, REDUCE_VLANES)[0])


def block_reduce_total(x: np.ndarray) -> float:
    """*total of a block_reduce_f32 dispatch (bit-exact target); within
    rounding of float(x.astype(float64).sum()), and equal to it on
    small-integer data."""
    return block_reduce_combine(block_reduce_partials(x))


def hbm_stream(src: np.ndarray) -> np.ndarray:
    """out = src (copy)."""
    return src.copy()
