"""CPU tests of bench.py's multi-process plumbing (gloo, world size 2): the
max-over-ranks time and summed units that make `value`, and the reference
arm's contract under torchrun (rank 0 prints one JSON line, other ranks exit
0 without work).  The LK path itself is replicas only -- no collective on the
data path -- so these are the only multi-rank pieces."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    import bench
    w, r, _ = bench.dist_setup()
    t, u = bench.gather_max_sum(w, 1.5 + r, 1000 * (r + 1))
    rows = bench.gather_rank_rows(w, {"rank": r, "p50_us": 2.0 + r})
    bench.barrier(w)
    q.put((r, t, u, [row["p50_us"] for row in rows]))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_gather_max_over_ranks_and_sum_of_units():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, t, u, p50s in out:
        assert t == 2.5 and u == 3000.0      # slowest rank's time, all ranks' units
        assert p50s == [2.0, 3.0]            # every rank's row on every rank, in rank order


def test_aggregate_is_units_over_slowest_rank():
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.aggregate([1.0, 2.0], [100, 300]) == 200.0


def test_reference_arm_under_torchrun_two_ranks():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "1", "--ref-rounds", "2",
           "--workers", "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0


def test_thread_driver_aggregate_is_rounds_over_slowest_thread():
    """bench.py --threads: whole-job tasks/s over the per-GPU host threads."""
    sys.path.insert(0, str(ROOT))
    import bench
    rows = [{"rounds": 1000, "elapsed_s": 0.5}, {"rounds": 1000, "elapsed_s": 1.0},
            {"rounds": 2000, "elapsed_s": 0.8}]
    v, t, u = bench.thread_driver_rows(rows)
    assert (v, t, u) == (4000.0, 1.0, 4000)


def test_threads_flag_refused_under_torchrun():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--threads", "--gpus", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0 and "--threads drives every GPU from one process" in r.stderr
