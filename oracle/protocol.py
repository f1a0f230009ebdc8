"""ORACLE (test infrastructure only): CPU restatement of the LK handshake.

Restates, in table form, /root/reference/pkg/src/persistkern/protocol.py:
  * word values                  protocol.py:31-45
  * decode_to_gpu                protocol.py:83-91
  * worker_step / complete_work  protocol.py:151-206
  * _host_write / _device_write  protocol.py:298-369
  * replay_trace                 protocol.py:372-392
Pinned by tests/golden/*.json (generated from the reference by
tests/golden/make_golden.py) and by the live reference when present.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Optional

INIT, FINISHED, WORKING, NOP, EXIT, WORK_BASE = 0, 1, 2, 4, 8, 16
WORD_MAX = 2**32 - 1
FROM_GPU = (INIT, FINISHED, WORKING, NOP)

# phases as short strings; the state is (phase, slot)
BOOT, IDLE, WORK, FIN, GONE = "booting", "idle", "working", "finished_pending_ack", "exited"


class Illegal(Exception):
    """The step is a protocol violation (protocol.py raises ProtocolViolation)."""


def command(word: int):
    """("nop",) / ("exit",) / ("work", slot); Illegal for any other word."""
    if word == NOP:
        return ("nop",)
    if word == EXIT:
        return ("exit",)
    if WORK_BASE <= word <= WORD_MAX:
        return ("work", word - WORK_BASE)
    raise Illegal(f"illegal to_gpu word {word}")


def step(phase: str, slot: Optional[int], word: int):
    """Return (phase', slot', publish|None, action) with action in
    {None, ("begin", slot), "exit"}; raise Illegal on a violation."""
    if phase == GONE:
        raise Illegal("worker stepped after exit")
    cmd = command(word)
    if cmd[0] == "exit" and phase != WORK:
        return GONE, None, None, "exit"
    if phase == BOOT:
        return IDLE, None, INIT, None
    if phase == IDLE:
        if cmd[0] == "nop":
            return IDLE, None, NOP, None
        return WORK, cmd[1], WORKING, ("begin", cmd[1])
    if phase == WORK:
        if cmd[0] == "work" and cmd[1] != slot:
            raise Illegal(f"work slot {cmd[1]} triggered while busy with slot {slot}")
        return WORK, slot, WORKING, None
    # FIN: awaiting the ack
    if cmd[0] == "nop":
        return IDLE, None, NOP, None
    if cmd[1] != slot:
        raise Illegal(f"work slot {cmd[1]} triggered before slot {slot} was acknowledged")
    return FIN, slot, FINISHED, None


def complete(phase: str, slot: Optional[int]):
    if phase != WORK:
        raise Illegal(f"completion signalled in phase {phase}")
    return FIN, slot, FINISHED, None


# ------------------------------------------------------------------ replay

@dataclass
class Cell:
    phase: Optional[str] = None   # None until the first device write is seen
    to_gpu: int = NOP
    from_gpu: int = NOP
    pending: bool = False
    work_writes: int = 0
    begins: int = 0


def _host(c: Cell, w: int) -> Optional[str]:
    if c.to_gpu == EXIT:
        return "host write after exit"
    if w == NOP:
        if c.from_gpu != FINISHED:
            return f"ack written while from_gpu={c.from_gpu}, not FINISHED"
        c.to_gpu = NOP
        return None
    if w == EXIT:
        if c.from_gpu == WORKING:
            return "exit written to a working cluster"
        if c.pending:
            return "exit would discard an undelivered work command"
        c.to_gpu = EXIT
        return None
    if WORK_BASE <= w <= WORD_MAX:
        if WORK_BASE <= c.to_gpu:
            return "trigger while busy: previous work command not consumed"
        if c.from_gpu not in (FINISHED, NOP):
            return f"work written while from_gpu={c.from_gpu}"
        c.to_gpu, c.pending = w, True
        c.work_writes += 1
        return None
    return f"illegal to_gpu word {w}"


def _device(c: Cell, w: int) -> Optional[str]:
    if w not in FROM_GPU:
        return f"illegal from_gpu word {w}"
    if c.phase is None:
        c.phase = IDLE
        if w == INIT:
            c.from_gpu = INIT
            return None
        c.from_gpu = NOP
    if c.phase == IDLE:
        if w == NOP and c.from_gpu == INIT:
            c.from_gpu = NOP
            return None
        if w == WORKING and c.to_gpu >= WORK_BASE and c.pending:
            c.phase, c.from_gpu, c.pending = WORK, WORKING, False
            c.begins += 1
            return None
        return f"word {w} not producible by an idle worker"
    if c.phase == WORK:
        if w == FINISHED:
            c.phase, c.from_gpu = FIN, FINISHED
            return None
        return f"word {w} not producible by a working worker"
    if w == NOP and c.to_gpu == NOP:
        c.phase, c.from_gpu = IDLE, NOP
        return None
    return f"word {w} not producible while awaiting ack"


@dataclass
class Replay:
    violation: Optional[tuple] = None          # (index, reason)
    cells: dict = field(default_factory=dict)

    def dispatch_counts(self) -> dict:
        return {i: (c.work_writes, c.begins) for i, c in self.cells.items()}


def replay(trace: Iterable) -> Replay:
    """Replay (side, sm_id, word) writes; stops at the first violation."""
    out = Replay()
    for index, (side, sm, word) in enumerate(trace):
        if sm < 0:
            out.violation = (index, f"negative sm_id {sm}")
            return out
        c = out.cells.setdefault(sm, Cell())
        if side == "H":
            why = _host(c, word)
        elif side == "D":
            why = _device(c, word)
        else:
            why = f"unknown side {side!r}"
        if why is not None:
            out.violation = (index, why)
            return out
    return out
