"""Phase timings and worker-mask helpers shared by the session classes.

Mirror of the helper half of persistkern.host
(/root/reference/pkg/src/persistkern/host.py:28-99).  On this runtime every
``cycles`` value is nanoseconds of host wall clock (as on the reference's
native backend, host.py:44).  Masks are Python ints, bit i = worker i; on
B200 a full mask is 148 bits wide and crosses the C ABI as little-endian
u64 words.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Optional

from .errors import UsageError

PHASE_INIT = "Init"
PHASE_ALLOC = "Alloc"
PHASE_COPYIN = "Copyin"
PHASE_TRIGGER = "Trigger"
PHASE_LAUNCH = "Launch"
PHASE_WAIT = "Wait"
PHASE_COPYOUT = "Copyout"
PHASE_DISPOSE = "Dispose"

MODEL_LK = "LK"
MODEL_BASELINE = "BASE"

_MASKED_PHASES = (PHASE_TRIGGER, PHASE_WAIT, PHASE_LAUNCH)


@dataclass(frozen=True)
class PhaseTiming:
    phase: str
    cycles: int        # nanoseconds on this runtime
    sm_mask: int = 0

    def __post_init__(self) -> None:
        if self.cycles < 0:
            raise ValueError("cycles must be nonnegative")
        if self.phase in _MASKED_PHASES and self.sm_mask == 0:
            raise ValueError(f"{self.phase} timing needs a nonempty sm mask")


_new = object.__new__


def _materialize(row: tuple) -> PhaseTiming:
    t = _new(PhaseTiming)
    d = t.__dict__
    d["phase"], d["cycles"], d["sm_mask"] = row
    return t


class TimingLog:
    """``session.timings``: the reference's ``list[PhaseTiming]``
    (P/native.py:99) as a sequence of PhaseTiming values.

    Rows are kept as plain (phase, cycles, sm_mask) tuples, which the garbage
    collector stops tracking after its first pass; a list of a million
    dataclass instances (plus their ``__dict__``s) is re-traversed by every
    older-generation collection, which cost more than the dispatch itself in
    long trigger/wait loops (tools/py_overhead.py).  Reading an entry builds
    an equal PhaseTiming."""

    __slots__ = ("_rows",)

    def __init__(self, items: Iterable[PhaseTiming] = ()) -> None:
        self._rows: list[tuple] = [(t.phase, t.cycles, t.sm_mask) for t in items]

    def append(self, t: PhaseTiming) -> None:
        self._rows.append((t.phase, t.cycles, t.sm_mask))

    def extend(self, items: Iterable[PhaseTiming]) -> None:
        for t in items:
            self.append(t)

    def clear(self) -> None:
        self._rows.clear()

    def pop(self, i: int = -1) -> PhaseTiming:
        return _materialize(self._rows.pop(i))

    def __len__(self) -> int:
        return len(self._rows)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [_materialize(r) for r in self._rows[i]]
        return _materialize(self._rows[i])

    def __iter__(self):
        for r in self._rows:
            yield _materialize(r)

    def __reversed__(self):
        for r in reversed(self._rows):
            yield _materialize(r)

    def __contains__(self, t) -> bool:
        return isinstance(t, PhaseTiming) and (t.phase, t.cycles, t.sm_mask) in self._rows

    def __eq__(self, other) -> bool:
        if isinstance(other, TimingLog):
            return self._rows == other._rows
        if isinstance(other, (list, tuple)):
            return list(self) == list(other)
        return NotImplemented

    __hash__ = None

    def __repr__(self) -> str:
        return repr(list(self))

    # the rest of list's mutable-sequence surface, for callers that edit the log
    def insert(self, i: int, t: PhaseTiming) -> None:
        self._rows.insert(i, (t.phase, t.cycles, t.sm_mask))

    def __setitem__(self, i, t) -> None:
        if isinstance(i, slice):
            self._rows[i] = [(x.phase, x.cycles, x.sm_mask) for x in t]
        else:
            self._rows[i] = (t.phase, t.cycles, t.sm_mask)

    def __delitem__(self, i) -> None:
        del self._rows[i]

    def index(self, t, *args) -> int:
        return self._rows.index((t.phase, t.cycles, t.sm_mask), *args)

    def count(self, t) -> int:
        return self._rows.count((t.phase, t.cycles, t.sm_mask)) if isinstance(t, PhaseTiming) else 0

    def copy(self) -> list:
        return list(self)


def full_mask(num_sms: int) -> int:
    return (1 << num_sms) - 1


def mask_of(sm_ids: Iterable[int]) -> int:
    m = 0
    for i in sm_ids:
        m |= 1 << i
    return m


def sms_in_mask(mask: int) -> list[int]:
    """Ascending ids of the set bits (host.py:66-73 semantics).  Scans the
    binary string instead of peeling bits off a big int: ~25x faster for a
    148-bit mask."""
    if mask <= 0:
        return []
    b = bin(mask)[:1:-1]
    return [i for i, c in enumerate(b) if c == "1"]


def _check_mask(mask: int, num_sms: int) -> list[int]:
    if mask <= 0:
        raise UsageError("sm mask must select at least one cluster")
    if mask >> num_sms:
        raise UsageError(f"sm mask {mask:#x} wider than {num_sms} clusters")
    return sms_in_mask(mask)


def timings_csv(rows, backend: Optional[str] = None) -> str:
    """``run_id,model,phase,sm_mask,cycles[,backend]`` rows (host.py:84-99)."""
    head = "run_id,model,phase,sm_mask,cycles" + (",backend" if backend is not None else "")
    lines = [head]
    for run_id, model, t in rows:
        cols = [str(run_id), model, t.phase, str(t.sm_mask), str(t.cycles)]
        if backend is not None:
            cols.append(backend)
        lines.append(",".join(cols))
    return "\n".join(lines) + "\n"


import collections.abc as _abc  # noqa: E402

_abc.MutableSequence.register(TimingLog)   # isinstance(session.timings, MutableSequence)
