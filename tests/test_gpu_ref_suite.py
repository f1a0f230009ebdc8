"""The reference's own test modules, unmodified, run against this package.

* /root/reference/pkg/tests/test_native.py -- every test, with
  persistkern.{native, protocol, host, errors, device} resolved to
  paper_2310_01212_b200's modules: the drop-in as a caller sees it.
* test_acceptance.py::test_criterion_8_native_stress (T/test_acceptance.py:
  187-223: 10,000 round-robin cycles on 4 workers, zero violations,
  exactly-once, median trigger < median spawn) with only persistkern.native
  replaced: the trace is validated by the REFERENCE's own protocol module.
* test_bench.py::test_native_backend_scenario_smoke (T/test_bench.py:196-
  203) on a fresh copy of the reference's own bench.py whose ``native`` is
  this package: the reference harness's unmodified "native" backend
  (_run_native_lk / _run_native_baseline, P/bench.py:218-241) drives the
  B200 session and the launch+sync baseline.

The modules are read from the reference tree when present (build container),
else from the unmodified copies __graft_entry__.build() stages under
oracle/_ref/tests/ (git-ignored; they travel to the GPU box with the repo).
"""
from __future__ import annotations

import dataclasses
import importlib.util
import sys
import types
from pathlib import Path

import pytest

from conftest import ROOT, reference_sys_path

pytestmark = pytest.mark.gpu

CANDIDATES = [Path("/root/reference/pkg/tests"), ROOT / "oracle" / "_ref" / "tests"]


def _source(name):
    for d in CANDIDATES:
        if (d / name).exists():
            return d / name
    return None


def _load(name, aliases):
    """Execute reference test module `name` with `aliases` (dotted name ->
    module) standing in for the persistkern modules it imports; sys.modules is
    restored afterwards (the loaded module keeps its bindings)."""
    path = _source(name)
    if path is None:
        pytest.skip(f"reference {name} not staged (run __graft_entry__.build())")
    ref = reference_sys_path()
    if ref is not None and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import persistkern as real_pkg
    saved = {k: sys.modules.get(k) for k in ["persistkern", *aliases]}
    fake = types.ModuleType("persistkern")
    fake.__path__ = real_pkg.__path__
    for attr in dir(real_pkg):
        if not attr.startswith("__"):
            setattr(fake, attr, getattr(real_pkg, attr))
    try:
        sys.modules["persistkern"] = fake
        for dotted, mod in aliases.items():
            sys.modules[dotted] = mod
            setattr(fake, dotted.split(".", 1)[1], mod)
        spec = importlib.util.spec_from_file_location(f"ref_{path.stem}", path)
        module = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(module)
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v
    return module


def _ours():
    from paper_2310_01212_b200 import device, errors, host, native, protocol
    return {"persistkern.native": native, "persistkern.protocol": protocol, "persistkern.host": host,
            "persistkern.errors": errors, "persistkern.device": device}


_NATIVE_TESTS = ["test_start_brings_workers_to_idle", "test_minimal_single_worker_session",
                 "test_boot_is_announced_in_the_trace", "test_zero_iteration_roundtrip_validates",
                 "test_multi_worker_stress_smoke", "test_full_mask_dispatch", "test_single_writer_word_sets",
                 "test_retrigger_busy_worker_rejected", "test_dispose_joins_every_thread",
                 "test_dispose_while_pending_rejected", "test_spin_until_times_out",
                 "test_trigger_latency_beats_thread_spawn", "test_descriptor_slot_locked_while_in_flight",
                 "test_timing_rows_carry_backend_column", "test_pinning_request_downgrades_gracefully",
                 "test_config_validation", "test_pure_spin_roundtrip"]


@pytest.fixture(scope="module")
def ref_native_tests():
    return _load("test_native.py", _ours())


def test_reference_suite_is_covered(ref_native_tests):
    """Every test function of the reference's test_native.py is in the list
    below (a new upstream test would show up here)."""
    found = sorted(n for n in dir(ref_native_tests) if n.startswith("test_"))
    assert found == sorted(_NATIVE_TESTS)


@pytest.mark.parametrize("name", _NATIVE_TESTS)
def test_reference_test_native(ref_native_tests, name):
    getattr(ref_native_tests, name)()


def _fresh_reference_module(name, aliases):
    """A new instance of reference module ``persistkern.<name>`` executed with
    ``aliases`` in sys.modules (so its ``from . import native`` binds this
    package's native); sys.modules is restored afterwards."""
    ref = reference_sys_path()
    if ref is not None and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import persistkern as real_pkg
    path = Path(real_pkg.__path__[0]) / f"{name}.py"
    dotted = f"persistkern.{name}"
    saved = {k: sys.modules.get(k) for k in [dotted, *aliases]}
    try:
        for k, mod in aliases.items():
            sys.modules[k] = mod
        spec = importlib.util.spec_from_file_location(dotted, path)
        module = importlib.util.module_from_spec(spec)
        module.__package__ = "persistkern"
        sys.modules[dotted] = module   # dataclasses resolve their module while the class is built
        spec.loader.exec_module(module)
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v
    return module


def test_reference_bench_native_backend_runs_on_b200():
    """The reference harness's own native backend, unmodified, on this
    package: Scenario(backend="native") -> run_scenario -> _run_native_lk /
    _run_native_baseline; the reference test asserts 5 samples per row and
    spawn (here: launch+sync) slower than trigger."""
    ours = _ours()
    bench = _fresh_reference_module("bench", {"persistkern.native": ours["persistkern.native"]})
    assert bench.native is ours["persistkern.native"]
    mod = _load("test_bench.py", {"persistkern.bench": bench})
    mod.test_native_backend_scenario_smoke()


def test_reference_cli_native_backend_on_b200_keeps_the_reference_behaviour():
    """`persistkern run --scenario table2-single-sm --backend native` through
    fresh copies of the reference's cli.py and bench.py bound to this
    package.  The scenario runs on the B200 (both models, 100 reps), then the
    reference's own compare step fails exactly as it does on the CPU: its
    native baseline emits no Dispose row (P/bench.py:233-241 vs 306), a
    reference defect SURVEY.md section 8(f) notes.  The drop-in reproduces
    it; the b200 backend (refharness, tests/test_gpu_refharness.py) adds
    the row and completes."""
    ours = _ours()
    bench = _fresh_reference_module("bench", {"persistkern.native": ours["persistkern.native"]})
    cli = _fresh_reference_module("cli", {"persistkern.bench": bench})
    assert cli.bench is bench and bench.native is ours["persistkern.native"]
    scenario = bench.builtin_scenarios()["table2-single-sm"]
    stats = bench.run_scenario(dataclasses.replace(scenario, backend="native"))
    assert stats.get("LK", "Wait").samples == scenario.reps
    assert stats.get("BASE", "Launch").samples == scenario.reps
    with pytest.raises(KeyError, match="BASE/Dispose"):
        cli.main(["run", "--scenario", "table2-single-sm", "--backend", "native"])


def test_reference_criterion_8_with_reference_validator():
    from paper_2310_01212_b200 import native
    acc = _load("test_acceptance.py", {"persistkern.native": native})
    assert acc.native is native and acc.protocol.__name__ == "persistkern.protocol"
    acc.test_criterion_8_native_stress()
