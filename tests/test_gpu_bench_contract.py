"""bench.py keeps the driver's JSON contract: one line on stdout with every
key the driver reads (metric, value, unit, n_gpus, steps, warmup,
ms_per_step, higher_is_better, scaling, vs_baseline, dtype, data, config,
e2e with its byte counts, gpu_launches, roofline, cpu_baseline, clocks),
and the headline latency keys last.  A short run with most extras off."""
from __future__ import annotations

import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_line_keeps_the_contract():
    cmd = [sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--rounds", "2000",
           "--full-rounds", "2000", "--e2e-rounds", "2000", "--base-rounds", "2000", "--pp-rounds", "2000",
           "--attrib-rounds", "2000", "--lazy-rounds", "2000", "--driver-rounds", "2000",
           "--payload-mib", "64", "--payload-reps", "3", "--config0-rounds", "200", "--cpu-budget-s", "3",
           "--no-interference", "--no-green", "--no-table2", "--no-zero-copy"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=280)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline",
              "cpu_baseline", "clocks", "per_rank"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 10_000
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["data"] == "synthetic"
    assert "workload" in d["config"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert 0.5 < d["roofline"]["frac"] < 1.2
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] >= 1
    keys = list(d)
    assert keys[-1] == "speedup_vs_launch_sync_p999" and "latency_us" in keys[-6:]


def test_bench_profiler_mode_skips_live_session_cuda_legs():
    """Under a profiler (detected from ncu's environment, faked here without
    any injection) bench.py keeps host descriptors and skips the legs that
    call CUDA while a session is resident; the line says it is not a bench
    value. profiles/r02_bench_launches_ncu.csv is this mode under real ncu."""
    import os
    env = dict(os.environ, NV_TPS_LAUNCH_TOKEN="test")
    cmd = [sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--rounds", "2000",
           "--full-rounds", "2000", "--e2e-rounds", "2000", "--base-rounds", "2000", "--attrib-rounds", "2000",
           "--driver-rounds", "2000", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=280, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert "profiled" in d and d["roofline"] is None and d["payload"] == {}
    for k in ("device_handling", "small_transfer", "pingpong_floor", "zero_copy", "lazy_ack", "interference"):
        assert k not in d, k
    assert d["value"] > 10_000 and d["gpu_launches"] >= 1
