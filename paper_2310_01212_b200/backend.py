"""The ``b200`` backend for the reference's scenario harness.

The reference selects executors in ``run_scenario`` by ``Scenario.backend``
(/root/reference/pkg/src/persistkern/bench.py:244-257) and runs the native
ones through ``_run_native_lk`` / ``_run_native_baseline`` (bench.py:218-241).
This module provides the B200 equivalents with the same inputs (any object
with the Scenario fields used there: ``reps``, ``cluster_count()``,
``mask()``, ``work()``) and returns per-phase sample lists that the
harness's own ``_aggregate`` turns into Table II/III rows (INTEGRATION.md
shows the six-line hook).

Differences from the reference's native runners, both deliberate:
* the baseline emits a ``Dispose`` row (stream + event teardown), so
  ``compare`` no longer raises ``KeyError: 'no stats for BASE/Dispose'`` on a
  native run (bench.py:233-241, 306 -- a reference bug);
* the baseline emits an ``Alloc`` row (stream/event creation), the
  counterpart of the sim baseline's (bench.py:190-200).
Timings are host nanoseconds, as on the reference's native backend
(host.py:44).
"""
from __future__ import annotations

import statistics
import time
from dataclasses import dataclass
from typing import Optional

from . import host, native

BACKEND_B200 = "b200"


@dataclass(frozen=True)
class PhaseStats:
    """Same fields as persistkern.bench.PhaseStats (bench.py:119-131)."""

    model: str
    phase: str
    avg: float
    worst: int
    best: int
    stddev: float
    samples: int

    def spread(self) -> float:
        return self.worst / self.avg if self.avg else 0.0


def aggregate(model: str, phase: str, samples: list[int]) -> PhaseStats:
    """persistkern.bench._aggregate (bench.py:151-159)."""
    return PhaseStats(model=model, phase=phase, avg=statistics.fmean(samples), worst=max(samples),
                      best=min(samples),
                      stddev=statistics.pstdev(samples) if len(samples) > 1 else 0.0,
                      samples=len(samples))


def _cfg(scenario, cfg: Optional[native.NativeConfig]) -> native.NativeConfig:
    n = scenario.cluster_count()
    if cfg is None:
        return native.NativeConfig(num_workers=n)
    return native.NativeConfig(**{**cfg.__dict__, "num_workers": n})


def lk_samples(scenario, cfg: Optional[native.NativeConfig] = None) -> dict[str, list[int]]:
    """``_run_native_lk`` on the B200 session: Init, reps x (Trigger, Wait), Dispose."""
    session, init = native.NativeSession.start(_cfg(scenario, cfg))
    try:
        mask, work = scenario.mask(), scenario.work()
        triggers, waits = [], []
        for _ in range(scenario.reps):
            triggers.append(session.trigger(mask, work).cycles)
            waits.append(session.wait(mask).cycles)
        dispose = session.dispose()
    finally:
        session.close()
    return {host.PHASE_INIT: [init.cycles], host.PHASE_TRIGGER: triggers, host.PHASE_WAIT: waits,
            host.PHASE_DISPOSE: [dispose.cycles]}


def baseline_samples(scenario, device: int = 0) -> dict[str, list[int]]:
    """``_run_native_baseline`` as cudaLaunchKernel + cudaStreamSynchronize of the
    same work function on a grid of ``popcount(mask)`` CTAs."""
    t0 = time.perf_counter_ns()
    base = native.LaunchSyncBaseline(device=device)
    alloc = time.perf_counter_ns() - t0
    grid = max(1, bin(scenario.mask()).count("1"))
    work = scenario.work()
    launches, waits = [], []
    try:
        for _ in range(scenario.reps):
            launches.append(base.launch(work, grid).cycles)
            waits.append(base.wait().cycles)
    finally:
        t1 = time.perf_counter_ns()
        base.close()
        dispose = time.perf_counter_ns() - t1
    return {host.PHASE_ALLOC: [alloc], host.PHASE_LAUNCH: launches, host.PHASE_WAIT: waits,
            host.PHASE_DISPOSE: [dispose]}


def run_b200(scenario, cfg: Optional[native.NativeConfig] = None, device: int = 0) -> list[PhaseStats]:
    """Both models of a Scenario on B200 hardware, as aggregated rows in the
    reference's order (LK rows first, then BASE, like run_scenario)."""
    rows: list[PhaseStats] = []
    models = scenario.models() if hasattr(scenario, "models") else [host.MODEL_LK, host.MODEL_BASELINE]
    for model in models:
        samples = lk_samples(scenario, cfg) if model == host.MODEL_LK else baseline_samples(scenario, device)
        rows += [aggregate(model, phase, s) for phase, s in samples.items()]
    return rows


def rows_csv(rows: list[PhaseStats]) -> str:
    """``model,phase,avg,worst,best,stddev,samples,backend`` (stats_csv body, bench.py:441-452)."""
    out = ["model,phase,avg,worst,best,stddev,samples,backend"]
    for r in rows:
        out.append(f"{r.model},{r.phase},{r.avg:.4f},{r.worst},{r.best},{r.stddev:.4f},{r.samples},"
                   f"{BACKEND_B200}")
    return "\n".join(out) + "\n"
