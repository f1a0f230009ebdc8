"""ORACLE (test infrastructure only): CPU port of the reference executor.

A thread-per-worker restatement of persistkern.native.NativeSession
(/root/reference/pkg/src/persistkern/native.py:82-299): N Python threads spin
on shared list cells under the GIL, stepping the oracle state machine
(oracle/protocol.py).  Used only as the timed CPU baseline on the GPU box
(`bench.py` cpu_baseline and `--impl reference`, kind "port"), where
/root/reference does not exist.  tests/test_oracle.py checks its traces
against the reference's validator and its timing against the live reference.

Departures from the reference, all opt-in: ``work_fn`` runs a payload
function on the worker thread (the reference's worker ignores payloads,
native.py:179-181), which is how the BASELINE "CPU reference" config's int32
vector add is executed.
"""
from __future__ import annotations

import itertools
import threading
import time
from typing import Callable, Optional

from . import protocol as P

PURE_SPIN = "pure_spin"
SPIN_THEN_YIELD = "spin_then_yield"


class PortError(Exception):
    pass


class CpuSession:
    def __init__(self, num_workers: int = 4, spin_strategy: str = SPIN_THEN_YIELD,
                 spin_yield_threshold: int = 10_000, record_trace: bool = False,
                 wait_timeout_s: float = 10.0,
                 work_fn: Optional[Callable[[int, int], None]] = None):
        self.n = num_workers
        self.yielding = spin_strategy == SPIN_THEN_YIELD
        self.yield_at = spin_yield_threshold
        self.record = record_trace
        self.timeout = wait_timeout_s
        self.work_fn = work_fn            # (worker_id, slot) -> None, runs on the worker
        self.to_gpu = [P.NOP] * num_workers
        self.from_gpu = [P.NOP] * num_workers
        self.phase = [P.BOOT] * num_workers
        self.errors: list = [None] * num_workers
        self.iterations: dict[int, int] = {}
        self.trace: list = []
        self._step = itertools.count()
        self.pending = 0
        self.pending_slots: dict[int, int] = {}
        self.threads: list[threading.Thread] = []

    # -- cells ---------------------------------------------------------------
    def _write(self, side: str, i: int, w: int) -> None:
        k = next(self._step)
        (self.to_gpu if side == "H" else self.from_gpu)[i] = w
        if self.record:
            self.trace.append((k, side, i, w))

    # -- worker ----------------------------------------------------------------
    def _worker(self, i: int) -> None:
        phase, slot, spins, settled = P.BOOT, None, 0, None
        cells = self.to_gpu
        try:
            while True:
                w = cells[i]
                if w == settled:
                    spins += 1
                    if self.yielding and spins >= self.yield_at:
                        spins = 0
                        time.sleep(0)
                    continue
                before = phase
                phase, slot, pub, act = P.step(phase, slot, w)
                moved = phase != before
                if pub is not None and pub != self.from_gpu[i]:
                    self._write("D", i, pub)
                    moved = True
                self.phase[i] = phase
                if act == "exit":
                    return
                if act is not None:                         # ("begin", slot)
                    n = self.iterations.get(slot, 0)
                    k = 0
                    while k < n:
                        k += 1
                    if self.work_fn is not None:
                        self.work_fn(i, slot)
                    phase, slot, pub, _ = P.complete(phase, slot)
                    self.phase[i] = phase
                    self._write("D", i, pub)
                    settled, spins = None, 0
                    continue
                settled = None if moved else w
                spins += 1
                if self.yielding and spins >= self.yield_at:
                    spins = 0
                    time.sleep(0)
        except BaseException as exc:
            self.errors[i] = exc
            self.phase[i] = P.GONE

    # -- host -------------------------------------------------------------------
    def start(self) -> int:
        t0 = time.perf_counter_ns()
        for i in range(self.n):
            th = threading.Thread(target=self._worker, args=(i,), daemon=True)
            self.threads.append(th)
            th.start()
        self._spin(lambda: all(p == P.IDLE for p in self.phase)
                   and all(w == P.NOP for w in self.from_gpu), "boot")
        return time.perf_counter_ns() - t0

    def _spin(self, cond, what: str) -> int:
        deadline = time.monotonic() + self.timeout
        spins = 0
        while True:
            if cond():
                return time.perf_counter_ns()
            for e in self.errors:
                if e is not None:
                    raise PortError(f"worker died: {e!r}")
            if time.monotonic() > deadline:
                raise PortError(f"{what} made no progress")
            spins += 1
            if self.yielding and spins >= self.yield_at:
                spins = 0
                time.sleep(0)

    def trigger(self, mask: int, slot: int, iterations: int = 0) -> int:
        ids = [i for i in range(self.n) if mask >> i & 1]
        if not ids or mask >> self.n:
            raise PortError("bad mask")
        if self.pending & mask or slot in self.pending_slots:
            raise PortError("busy")
        if any(self.from_gpu[i] != P.NOP for i in ids):
            raise PortError("not idle")
        t0 = time.perf_counter_ns()
        self.iterations[slot] = iterations
        for i in ids:
            self._write("H", i, P.WORK_BASE + slot)
        dt = time.perf_counter_ns() - t0
        self.pending |= mask
        self.pending_slots[slot] = mask
        return dt

    def wait(self, mask: int) -> int:
        ids = [i for i in range(self.n) if mask >> i & 1]
        t0 = time.perf_counter_ns()
        done = self._spin(lambda: all(self.from_gpu[i] == P.FINISHED for i in ids), "finish")
        for i in ids:
            self._write("H", i, P.NOP)
        self._spin(lambda: all(self.from_gpu[i] == P.NOP for i in ids), "ack")
        self.pending &= ~mask
        for s in list(self.pending_slots):
            left = self.pending_slots[s] & ~mask
            if left:
                self.pending_slots[s] = left
            else:
                del self.pending_slots[s]
        return done - t0

    def dispose(self) -> int:
        if self.pending:
            raise PortError("dispose while busy")
        t0 = time.perf_counter_ns()
        for i in range(self.n):
            self._write("H", i, P.EXIT)
        for th in self.threads:
            th.join(timeout=self.timeout)
            if th.is_alive():
                raise PortError("worker did not exit")
        return time.perf_counter_ns() - t0

    def writes(self) -> list:
        return [(s, i, w) for _, s, i, w in sorted(self.trace)]
