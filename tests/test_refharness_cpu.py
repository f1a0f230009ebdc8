"""The b200 backend patched into the reference's own scenario harness
(paper_2310_01212_b200.refharness): validation, CLI parsing and the sim path
are checked here without a GPU; tests/test_gpu_refharness.py runs it."""
from __future__ import annotations

import pytest

from paper_2310_01212_b200 import refharness


@pytest.fixture
def patched(refpkg):
    bench, cli = refpkg["bench"], refpkg["cli"]
    refharness.install(bench, cli)
    yield bench, cli
    refharness.uninstall()


def test_b200_backend_is_accepted_and_others_still_validated(patched):
    bench, _ = patched
    s = bench.Scenario(name="x", backend="b200")
    assert s.backend == "b200"
    from persistkern.errors import UsageError
    with pytest.raises(UsageError):
        bench.Scenario(name="x", backend="cuda")
    with pytest.raises(UsageError):
        bench.Scenario(name="x", backend="b200", reps=0)   # the reference's other rules still apply


def test_cli_offers_b200(patched):
    _, cli = patched
    args = cli.build_parser().parse_args(["run", "--scenario", "table2-single-sm", "--backend", "b200"])
    assert args.backend == "b200"


def test_sim_backend_unchanged(patched):
    bench, _ = patched
    import dataclasses
    s = dataclasses.replace(bench.builtin_scenarios()["table2-single-sm"], reps=3)
    stats = bench.run_scenario(s)
    assert stats.has("LK", "Trigger") and stats.has("BASE", "Launch")


def test_uninstall_restores(refpkg):
    bench, cli = refpkg["bench"], refpkg["cli"]
    post, run, build = bench.Scenario.__post_init__, bench.run_scenario, cli.build_parser
    refharness.install(bench, cli)
    assert bench.run_scenario is not run
    refharness.uninstall()
    assert bench.Scenario.__post_init__ is post and bench.run_scenario is run and cli.build_parser is build
