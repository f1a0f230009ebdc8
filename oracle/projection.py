"""ORACLE (test infrastructure only): expected per-worker write projections.

For a native session that boots, runs a sequence of dispatches and disposes,
every worker's own sub-sequence of value-changing writes is fixed by the
handshake (persistkern.protocol.worker_step + NativeSession.trigger/wait/
dispose, protocol.py:151-206, native.py:208-295):

    D0 D4  ( H[16+slot] D2 D1 H4 D4 )*  H8

(verified against the reference's own NativeSession, tests/golden).
"""
from __future__ import annotations

from . import protocol as P


def expected_projection(slots: list[int], disposed: bool = True) -> list[tuple[str, int]]:
    out = [("D", P.INIT), ("D", P.NOP)]
    for s in slots:
        out += [("H", P.WORK_BASE + s), ("D", P.WORKING), ("D", P.FINISHED), ("H", P.NOP), ("D", P.NOP)]
    if disposed:
        out.append(("H", P.EXIT))
    return out


def projections(writes, num_workers: int) -> dict[int, list[tuple[str, int]]]:
    out: dict[int, list] = {i: [] for i in range(num_workers)}
    for side, sm, word in writes:
        out.setdefault(sm, []).append((side, word))
    return out


def program_slots(program, num_workers: int) -> dict[int, list[int]]:
    """program: [(mask, slot), ...] in dispatch order -> per-worker slot list."""
    per: dict[int, list[int]] = {i: [] for i in range(num_workers)}
    for mask, slot in program:
        for i in range(num_workers):
            if mask >> i & 1:
                per[i].append(slot)
    return per
