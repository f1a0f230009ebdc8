"""Run the reference's own scenario harness on B200 hardware.

The reference picks an executor in ``run_scenario`` by ``Scenario.backend``
(/root/reference/pkg/src/persistkern/bench.py:244-257, validated in
``Scenario.__post_init__`` at bench.py:77-78) and exposes the choice on the
CLI as ``--backend`` (cli.py:264).  :func:`install` adds a third backend,
``"b200"``, to an imported, unmodified ``persistkern`` package at run time:

* ``Scenario.__post_init__`` accepts ``backend="b200"`` (every other rule of
  the original validation still runs);
* ``run_scenario`` sends b200 scenarios to :func:`backend.run_b200` -- the
  LK session and the launch+sync baseline on the GPU -- and returns the
  reference's own ``RunStats`` of the reference's own ``PhaseStats`` rows, so
  ``compare``, ``render_table``, ``stats_csv`` and ``evaluate_scenario`` run
  unchanged on them;
* ``cli.build_parser`` offers ``b200`` among the ``--backend`` choices, so
  ``persistkern run --scenario table2-full-gpu --backend b200`` works.

No reference file is edited; :func:`uninstall` restores the originals.
"""
from __future__ import annotations

import argparse
import dataclasses
from typing import Optional

from . import backend as _backend

B200 = _backend.BACKEND_B200
_SAVED: dict = {}


def _stats_rows(bench, rows):
    return [bench.PhaseStats(model=r.model, phase=r.phase, avg=r.avg, worst=r.worst, best=r.best, stddev=r.stddev,
                             samples=r.samples) for r in rows]


def install(bench, cli=None, *, num_sms: Optional[int] = None, device: int = 0) -> None:
    """Patch the reference modules ``bench`` (persistkern.bench) and ``cli``
    (persistkern.cli) in place.  ``num_sms``: run b200 scenarios on this many
    workers instead of the scenario's own count (e.g. 148, the whole B200;
    the builtin Table II scenarios model the paper's 16-SM GTX980)."""
    if "bench" in _SAVED:
        return
    _SAVED["bench"] = (bench, bench.Scenario.__post_init__, bench.run_scenario)
    orig_post, orig_run = bench.Scenario.__post_init__, bench.run_scenario

    def post_init(self):
        if self.backend != B200:
            return orig_post(self)
        # validate everything else exactly as the reference does
        object.__setattr__(self, "backend", bench.BACKEND_NATIVE)
        try:
            orig_post(self)
        finally:
            object.__setattr__(self, "backend", B200)

    def run_scenario(s):
        if s.backend != B200:
            return orig_run(s)
        scn = s if num_sms is None else dataclasses.replace(s, num_sms=num_sms, device=None)
        stats = bench.RunStats(s)
        stats.rows.extend(_stats_rows(bench, _backend.run_b200(scn, device=device)))
        return stats

    bench.Scenario.__post_init__ = post_init
    bench.run_scenario = run_scenario

    if cli is not None:
        _SAVED["cli"] = (cli, cli.build_parser)
        orig_build = cli.build_parser

        def build_parser():
            parser = orig_build()
            for act in parser._actions:
                if isinstance(act, argparse._SubParsersAction):
                    for a in act.choices["run"]._actions:
                        if a.dest == "backend" and a.choices is not None and B200 not in a.choices:
                            a.choices = list(a.choices) + [B200]
            return parser

        cli.build_parser = build_parser


def uninstall() -> None:
    if "bench" in _SAVED:
        bench, post, run = _SAVED.pop("bench")
        bench.Scenario.__post_init__ = post
        bench.run_scenario = run
    if "cli" in _SAVED:
        cli, build = _SAVED.pop("cli")
        cli.build_parser = build
