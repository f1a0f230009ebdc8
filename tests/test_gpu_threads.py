"""configs[4] in the north star's form (bench.py --threads): one session per
visible GPU in ONE process, one NUMA-pinned host thread each.  On a 1-GPU box
this runs one thread; the aggregation rule is covered on CPU
(tests/test_bench_dist.py)."""
from __future__ import annotations

import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_threads_arm_runs_every_visible_gpu():
    from paper_2310_01212_b200 import native
    out = subprocess.run([sys.executable, "bench.py", "--threads", "--steps", "3", "--warmup", "1",
                          "--rounds", "2000"], cwd=ROOT, capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert "error" not in line, line
    assert line["n_gpus"] == native.device_count() == len(line["per_gpu"])
    assert all(r["rounds"] == 6000 and r["trigger_to_done"]["p50_us"] > 0 for r in line["per_gpu"])
    assert line["value"] > 10_000
    assert len({r["core"] for r in line["per_gpu"]}) == len(line["per_gpu"])   # one core per thread
