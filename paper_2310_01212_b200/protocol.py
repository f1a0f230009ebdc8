"""Mailbox wire words, the worker state machine and trace tooling.

API mirror of persistkern.protocol
(/root/reference/pkg/src/persistkern/protocol.py) for the B200 runtime:

* word values and host commands (protocol.py:31-98) are plain constants;
* ``worker_step`` / ``complete_work`` (protocol.py:151-206) call the host build
  of the *same* state machine the persistent kernel runs
  (csrc/lk_protocol.cuh via lk_protocol_step), so the golden transition table
  checks the device logic itself;
* ``replay_trace`` / ``validate_trace`` (protocol.py:372-398) run the native
  replay in csrc/lk_validate.cpp, fast enough for million-record GPU traces;
* the trace file format (protocol.py:401-432) is unchanged.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum
from typing import Iterable, Optional, Sequence, Union

import numpy as np

from . import _lib
from .errors import ProtocolViolation

WORD_BITS = 32
WORD_MAX = (1 << WORD_BITS) - 1
WORD_SIZE_BYTES = 4

INIT, FINISHED, WORKING, NOP = 0, 1, 2, 4      # from_gpu
EXIT, WORK_BASE = 8, 16                        # to_gpu (plus NOP)
FROM_GPU_WORDS = frozenset({INIT, FINISHED, WORKING, NOP})
MAX_SLOT = WORD_MAX - WORK_BASE

HOST_SIDE, DEVICE_SIDE = "H", "D"


@dataclass(frozen=True)
class Nop:
    """Idle / acknowledge command."""


@dataclass(frozen=True)
class Exit:
    """Leave the spin loop for good."""


@dataclass(frozen=True)
class Work:
    """Run the descriptor registered under ``slot``."""

    slot: int


HostCommand = Union[Nop, Exit, Work]


def encode_to_gpu(cmd: HostCommand) -> int:
    if isinstance(cmd, Work):
        if not 0 <= cmd.slot <= MAX_SLOT:
            raise ProtocolViolation(
                f"work slot {cmd.slot} does not fit in a {WORD_BITS}-bit word", word=None)
        return WORK_BASE + cmd.slot
    if isinstance(cmd, Nop):
        return NOP
    if isinstance(cmd, Exit):
        return EXIT
    raise TypeError(f"not a host command: {cmd!r}")


def is_work_word(word: int) -> bool:
    return WORK_BASE <= word <= WORD_MAX


def decode_to_gpu(word: int) -> HostCommand:
    if is_work_word(word):
        return Work(word - WORK_BASE)
    if word == NOP:
        return Nop()
    if word == EXIT:
        return Exit()
    raise ProtocolViolation(f"illegal to_gpu word {word}", word=word)


class Phase(Enum):
    BOOTING = "booting"
    IDLE = "idle"
    WORKING = "working"
    FINISHED_PENDING_ACK = "finished_pending_ack"
    EXITED = "exited"


# device phase codes (include/lk.h LK_PHASE_*) <-> Phase
PHASE_OF_CODE = {0: Phase.BOOTING, 1: Phase.IDLE, 2: Phase.WORKING,
                 3: Phase.FINISHED_PENDING_ACK, 4: Phase.EXITED}
CODE_OF_PHASE = {v: k for k, v in PHASE_OF_CODE.items()}


@dataclass(frozen=True)
class WorkerState:
    phase: Phase = Phase.BOOTING
    slot: Optional[int] = None

    def __post_init__(self) -> None:
        busy = self.phase in (Phase.WORKING, Phase.FINISHED_PENDING_ACK)
        if busy != (self.slot is not None):
            raise ValueError(f"{self.phase} {'requires' if busy else 'must not carry'} a slot")


@dataclass(frozen=True)
class BeginWork:
    slot: int


@dataclass(frozen=True)
class ExitLoop:
    pass


Action = Union[BeginWork, ExitLoop, None]


@dataclass(frozen=True)
class StepResult:
    state: WorkerState
    publish: Optional[int]
    action: Action


_NO_PUBLISH = 0xFFFFFFFF


def _native_state(state: WorkerState):
    return C.c_uint32(CODE_OF_PHASE[state.phase]), C.c_uint32(state.slot or 0)


def _result(ph: C.c_uint32, sl: C.c_uint32, pub: C.c_uint32, act: int) -> StepResult:
    phase = PHASE_OF_CODE[ph.value]
    busy = phase in (Phase.WORKING, Phase.FINISHED_PENDING_ACK)
    state = WorkerState(phase, sl.value if busy else None)
    action: Action = None
    if act == 1:
        action = BeginWork(sl.value)
    elif act == 2:
        action = ExitLoop()
    return StepResult(state, None if pub.value == _NO_PUBLISH else pub.value, action)


def worker_step(state: WorkerState, observed: int) -> StepResult:
    """One poll of the device worker loop, run through the kernel's own logic."""
    if not 0 <= observed <= WORD_MAX:
        raise ProtocolViolation(f"illegal to_gpu word {observed}", word=observed)
    lib = _lib.load()
    ph, sl = _native_state(state)
    pub, act, werr = C.c_uint32(), C.c_uint32(), C.c_uint32()
    rc = lib.lk_protocol_step(C.byref(ph), C.byref(sl), observed, C.byref(pub), C.byref(act),
                              C.byref(werr))
    if rc != 0:
        raise ProtocolViolation(f"{_lib.WERR_NAMES.get(werr.value, 'violation')} "
                                f"(phase {state.phase.value}, word {observed})", word=observed)
    return _result(ph, sl, pub, act.value)


def complete_work(state: WorkerState) -> StepResult:
    lib = _lib.load()
    ph, sl = _native_state(state)
    pub, werr = C.c_uint32(), C.c_uint32()
    rc = lib.lk_protocol_complete(C.byref(ph), C.byref(sl), C.byref(pub), C.byref(werr))
    if rc != 0:
        raise ProtocolViolation(f"completion signalled in phase {state.phase}")
    return _result(ph, sl, pub, 0)


# ---------------------------------------------------------------- mailboxes

@dataclass
class MailboxPair:
    sm_id: int
    to_gpu: int = NOP
    from_gpu: int = NOP


@dataclass
class Mailboard:
    entries: list

    @classmethod
    def create(cls, num_sms: int) -> "Mailboard":
        return cls([MailboxPair(sm_id=i) for i in range(num_sms)])

    def __len__(self) -> int:
        return len(self.entries)

    def __getitem__(self, sm_id: int) -> MailboxPair:
        return self.entries[sm_id]

    def serialized_bytes(self) -> int:
        return board_bytes(len(self.entries))


def board_bytes(num_sms: int) -> int:
    """Protocol payload of a board: one word per direction per worker."""
    return 2 * WORD_SIZE_BYTES * num_sms


# ---------------------------------------------------------------- traces

@dataclass(frozen=True)
class TraceRecord:
    step: int
    side: str
    sm_id: int
    word: int

    def to_line(self) -> str:
        return f"{self.step},{self.side},{self.sm_id},{self.word}"


@dataclass(frozen=True)
class Violation:
    index: int
    reason: str

    def __str__(self) -> str:
        return f"violation at index {self.index}: {self.reason}"


@dataclass
class ReplayState:
    counts: dict

    def dispatch_counts(self) -> dict:
        """Per worker: (host WORK writes, device begin transitions)."""
        return dict(self.counts)


def _as_arrays(trace):
    if isinstance(trace, tuple) and len(trace) == 3 and isinstance(trace[0], np.ndarray):
        side, sm, word = trace
        return (np.ascontiguousarray(side, dtype=np.uint32), np.ascontiguousarray(sm, dtype=np.int64),
                np.ascontiguousarray(word, dtype=np.uint32), None)
    rows = list(trace)
    n = len(rows)
    side = np.empty(n, dtype=np.uint32)
    sm = np.empty(n, dtype=np.int64)
    word = np.empty(n, dtype=np.uint32)
    words_raw = []
    for i, (s, m, w) in enumerate(rows):
        side[i] = ord(s[0]) if isinstance(s, str) and len(s) == 1 else 0
        sm[i] = m
        words_raw.append(w)
        word[i] = w if 0 <= w <= WORD_MAX else 3   # out-of-range: illegal either way
    return side, sm, word, rows


def replay_trace(trace: Iterable) -> tuple[Optional[Violation], ReplayState]:
    """Replay (side, sm_id, word) writes natively; first violation + counts.

    ``trace`` is an iterable of tuples or a (side_u32, sm_i64, word_u32) tuple
    of numpy arrays (side as ord('H') / ord('D')).
    """
    side, sm, word, rows = _as_arrays(trace)
    lib = _lib.load()
    bad = C.c_int64(-1)
    reason = C.create_string_buffer(256)
    maxw = max(1, len(np.unique(sm))) if len(sm) else 1
    counts = np.zeros(3 * maxw, dtype=np.uint64)
    nworkers = C.c_uint32()
    _lib.check(lib.lk_validate_trace(side.ctypes.data, sm.ctypes.data, word.ctypes.data, len(side),
                                     C.byref(bad), reason, 256, counts.ctypes.data_as(_lib.PU64), maxw,
                                     C.byref(nworkers)))
    if rows is not None and bad.value >= 0:
        s = rows[bad.value][0]
        if not (isinstance(s, str) and len(s) == 1):
            reason = C.create_string_buffer(f"unknown side {s!r}".encode())
    got = {int(counts[3 * k]): (int(counts[3 * k + 1]), int(counts[3 * k + 2]))
           for k in range(nworkers.value)}
    violation = None if bad.value < 0 else Violation(bad.value, reason.value.decode())
    return violation, ReplayState(got)


def validate_trace(trace: Iterable) -> Optional[Violation]:
    return replay_trace(trace)[0]


def format_trace(records: Sequence[TraceRecord]) -> str:
    return "".join(r.to_line() + "\n" for r in records)


def parse_trace(text: str) -> list[TraceRecord]:
    out: list[TraceRecord] = []
    prev = -1
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        fields = line.split(",")
        if len(fields) != 4:
            raise ValueError(f"line {lineno}: expected 4 fields, got {len(fields)}")
        try:
            step, sm_id, word = int(fields[0]), int(fields[2]), int(fields[3])
        except ValueError as exc:
            raise ValueError(f"line {lineno}: {exc}") from None
        side = fields[1].strip()
        if side not in (HOST_SIDE, DEVICE_SIDE):
            raise ValueError(f"line {lineno}: side must be H or D, got {side!r}")
        if step <= prev:
            raise ValueError(f"line {lineno}: step {step} not increasing")
        prev = step
        out.append(TraceRecord(step, side, sm_id, word))
    return out
