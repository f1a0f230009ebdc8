"""Benchmark: LK trigger->done round trips on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lk|reference]

Workload (BASELINE.json configs[1]): one persistent CTA on each of the 148
SMs, empty task, round-robin single-worker dispatch ``mask = 1 << (k % 148)``.
A *step* is ``--rounds`` (default 20,000) closed-loop trigger+wait round
trips driven from C (lk_bench_roundtrip); the default 50 steps are the 1e6
rounds the config names.  ``value`` = round trips (tasks) per second over the
whole job (sum over ranks / max-over-ranks time).  Latency is host-observed
by definition (trigger start -> FINISHED seen, native.py:256-259), so it is
timed with CLOCK_MONOTONIC per round.  A device-wide synchronize cannot bracket
the region: the persistent kernel stays resident, so cudaDeviceSynchronize (and
torch.cuda.synchronize) would never return.  The C loop is itself synchronous
(every round ends with the workers' NOP observed on the host), and ranks
barrier (gloo, CPU-only) on both sides.

Extra objects on the JSON line: latency percentiles and jitter, the
cudaLaunchKernel+cudaStreamSynchronize baseline and the cheapest
conventional flows (empty kernel, stream query, CUDA graph, spin scheduling),
the raw PCIe ping-pong floor, the full-148-worker variant, payload HBM GB/s
(SAXPY / block reduce 1-64 MiB, L2-cold by buffer rotation, device
globaltimer spans) on the payload session and on the DIRECT one, the roofline
of the dominant payload kernel, zero-copy small transfers against cudaMemcpy
(and the paper's full-board mailbox workaround), the interference tests,
Table II through the reference's scenarios, the tail attribution, and the CPU
baseline (the unmodified reference executor, timed on this host).  The
latency headline and the speed-up ratios are the last keys of the line.

Multi-GPU (torchrun): one independent LK instance per GPU, host thread pinned
to the GPU's NUMA-local cores; "replicas only", no collective on the path;
every rank's p50/p99.9 in `per_rank`.  `--threads`: the same in one process,
one NUMA-pinned host thread per visible GPU.

Under ncu (`ncu --metrics gpu__time_duration.sum python bench.py ...`) the
same command runs for its launch list: the session keeps its descriptors in
mapped host memory and the legs that make CUDA calls while a session is
resident are skipped; the line is marked "profiled" and is not a bench value.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MEASURED_PEAKS = ROOT / "MEASURED_PEAKS.json"
SM_MAX_GHZ = 1.965
FALLBACK_HBM_GBS = 6650.0
L2_BYTES = 126 * 1024 * 1024


def pct(a, q):
    return float(np.percentile(np.asarray(a, dtype=np.float64), q))


def lat_summary(ns):
    ns = np.asarray(ns, dtype=np.float64)
    p50, p999 = pct(ns, 50), pct(ns, 99.9)
    return {"p50_us": round(p50 / 1e3, 3), "p99_us": round(pct(ns, 99) / 1e3, 3),
            "p99.9_us": round(p999 / 1e3, 3), "max_us": round(float(ns.max()) / 1e3, 3),
            "mean_us": round(float(ns.mean()) / 1e3, 3), "jitter_us": round((p999 - p50) / 1e3, 3),
            "n": int(ns.size)}


def hbm_peak():
    try:
        j = json.loads(MEASURED_PEAKS.read_text())
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int, avoid_core=None):
        self.device = device
        self.proc = None
        self.avoid = avoid_core

    def _away(self):
        # the sampler must not inherit the pinned spinning core: its wakeups
        # would preempt the timed host thread (rescheduling IPIs, slow rounds)
        if self.avoid is None:
            return
        try:
            cores = set(_ALLOWED_CORES or os.sched_getaffinity(0)) - {self.avoid}
            if cores:
                os.sched_setaffinity(0, cores)
        except OSError:
            pass

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
                preexec_fn=self._away)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (getattr(self, "out", "") or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


class CoreNoise:
    """Interrupts delivered to one CPU and its steal/irq time (/proc) across
    a region: the host-side evidence for latency tails (a 4-us slow round on
    a pinned spinning core is an interrupt or a vCPU preemption)."""

    def __init__(self, cpu):
        self.cpu = cpu

    @staticmethod
    def _irqs(cpu):
        out = {}
        try:
            lines = Path("/proc/interrupts").read_text().splitlines()
            cols = lines[0].split()
            idx = cols.index(f"CPU{cpu}")
            for ln in lines[1:]:
                f = ln.split()
                if len(f) > idx + 1 and f[0].endswith(":"):
                    try:
                        out[f[0][:-1]] = int(f[idx + 1])
                    except ValueError:
                        pass
        except Exception:
            pass
        return out

    @staticmethod
    def _stat(cpu):
        try:
            for ln in Path("/proc/stat").read_text().splitlines():
                f = ln.split()
                if f[0] == f"cpu{cpu}":
                    v = [int(x) for x in f[1:]]
                    return {"irq": v[5], "softirq": v[6], "steal": v[7]}
        except Exception:
            pass
        return {}

    def __enter__(self):
        self.i0, self.s0, self.t0 = self._irqs(self.cpu), self._stat(self.cpu), time.perf_counter()
        return self

    def __exit__(self, *exc):
        self.i1, self.s1, self.t1 = self._irqs(self.cpu), self._stat(self.cpu), time.perf_counter()

    def summary(self, lat_ns=None, p50_ns=None):
        d = {k: self.i1.get(k, 0) - v for k, v in self.i0.items()}
        d = {k: v for k, v in d.items() if v}
        tick = os.sysconf("SC_CLK_TCK") if hasattr(os, "sysconf") else 100
        out = {"cpu": self.cpu, "seconds": round(self.t1 - self.t0, 3), "irqs_total": sum(d.values()),
               "irqs_by_source": dict(sorted(d.items(), key=lambda kv: -kv[1])[:8]),
               "steal_ms": round(1e3 * (self.s1.get("steal", 0) - self.s0.get("steal", 0)) / tick, 1),
               "irq_ms": round(1e3 * (self.s1.get("irq", 0) - self.s0.get("irq", 0)) / tick, 1),
               "softirq_ms": round(1e3 * (self.s1.get("softirq", 0) - self.s0.get("softirq", 0)) / tick, 1)}
        if lat_ns is not None and p50_ns is not None:
            a = np.asarray(lat_ns, dtype=np.float64)
            out["slow_rounds_gt_p50_plus_2us"] = int((a > p50_ns + 2000).sum())
            out["rounds"] = int(a.size)
        return out


# ----------------------------------------------------------------------------- dist

def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")   # CPU collectives only: no kernels beside the resident LK
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def gather_max_sum(world, t_s, units):
    if world == 1:
        return t_s, units
    import torch
    import torch.distributed as dist
    t = torch.tensor([t_s], dtype=torch.float64)
    u = torch.tensor([units], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


def gather_rank_rows(world, row):
    """Every rank's small summary dict, on every rank (gloo all_gather_object);
    [row] at world size 1."""
    if world == 1:
        return [row]
    import torch.distributed as dist
    rows = [None] * world
    dist.all_gather_object(rows, row)
    return rows


def aggregate(rank_times, rank_units):
    """Whole-job throughput: total units / slowest rank's time."""
    return sum(rank_units) / max(rank_times)


# ----------------------------------------------------------------------------- CPU baseline

MIN_TIMED_ROUNDS = 20


def _over_budget(t_start, budget_s, k, warmup, timed):
    """Stop a bounded CPU sample once its time budget is spent, but never
    before MIN_TIMED_ROUNDS timed rounds (a small budget may be spent in the
    warm-up alone)."""
    if timed >= MIN_TIMED_ROUNDS and time.perf_counter() - t_start > budget_s:
        return True
    return False


def cpu_baseline_config0(num_workers=4, rounds=1000, warmup=50, n=65536, threshold=10_000, budget_s=30.0):
    """BASELINE config 0 on this host's cores: 4 workers, int32 vector add of
    64 Ki elements run on the worker thread, round-robin masks, the given
    spin_yield_threshold.  Runs the unmodified reference executor
    (baseline/_ref) with its descriptor table swapped for a dict whose lookup
    (native.py:180, on the worker thread) performs the vector add -- a harness
    shim, no reference edit; else the oracle port.  Returns (tasks/s, ns
    latencies, kind).  Call with the process's full CPU affinity: the
    reference's worker threads inherit it."""
    from oracle import work as W
    a = np.random.default_rng(0).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    b = np.random.default_rng(1).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    out = np.empty(n, np.int32)

    Exe = reference_executor()
    if Exe.kind == "reference":
        from persistkern import native as ref_native
        from persistkern.device import WorkDescriptor as RefWork

        class _PayloadTable(dict):
            def __getitem__(self, slot):
                np.copyto(out, W.vector_add_i32(a, b))
                return dict.__getitem__(self, slot)

        rs, _ = ref_native.NativeSession.start(
            ref_native.NativeConfig(num_workers=num_workers, spin_yield_threshold=threshold))
        rs.descriptors = _PayloadTable()
        rw = RefWork(slot=0, iterations=0)

        class _S:
            def trigger(self, m, _slot):
                rs.trigger(m, rw)

            def wait(self, m):
                rs.wait(m)

            def dispose(self):
                rs.dispose()
        s = _S()
    else:
        from oracle.cpu_session import CpuSession

        def work_fn(i, slot):
            np.copyto(out, W.vector_add_i32(a, b))
        s = CpuSession(num_workers=num_workers, spin_yield_threshold=threshold, work_fn=work_fn)
        s.start()
    lat = []
    t_start = time.perf_counter()
    for k in range(warmup + rounds):
        m = 1 << (k % num_workers)
        t0 = time.perf_counter_ns()
        s.trigger(m, 0)
        s.wait(m)
        if k >= warmup:
            lat.append(time.perf_counter_ns() - t0)
        if _over_budget(t_start, budget_s, k, warmup, len(lat)):
            break
    s.dispose()
    assert np.array_equal(out, W.vector_add_i32(a, b))
    tot = sum(lat) / 1e9
    return len(lat) / tot, lat, Exe.kind


def cpu_spawn_baseline_config0(rounds=1000, warmup=50, n=65536, budget_s=10.0):
    """The reference's own conventional flow on configs[0]'s task:
    persistkern.native.ThreadSpawnBaseline.launch/wait (P/native.py:304-331),
    one fresh thread per task.  Its target _busy_loop is looked up in the
    module at launch time, so it is swapped for the vector add for the run
    (harness shim, restored after; no reference edit).  Returns (tasks/s, ns
    latencies) or None without baseline/_ref."""
    from oracle import work as W
    if reference_executor().kind != "reference":
        return None
    from persistkern import native as ref_native
    from persistkern.device import WorkDescriptor as RefWork
    a = np.random.default_rng(0).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    b = np.random.default_rng(1).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    out = np.empty(n, np.int32)
    orig = ref_native._busy_loop

    def task(_iterations):
        np.copyto(out, W.vector_add_i32(a, b))
        return 0
    ref_native._busy_loop = task
    try:
        base = ref_native.ThreadSpawnBaseline()
        w = RefWork(slot=0, iterations=0)
        lat = []
        t_start = time.perf_counter()
        for k in range(warmup + rounds):
            t0 = time.perf_counter_ns()
            base.launch(w)
            base.wait()
            if k >= warmup:
                lat.append(time.perf_counter_ns() - t0)
            if _over_budget(t_start, budget_s, k, warmup, len(lat)):
                break
    finally:
        ref_native._busy_loop = orig
    assert np.array_equal(out, W.vector_add_i32(a, b))
    return len(lat) / (sum(lat) / 1e9), lat


REF_DIR = ROOT / "baseline" / "_ref"


def reference_executor():
    """The unmodified reference executor: persistkern.native from baseline/_ref
    (pip-installed from /root/reference, travels to the GPU box) -> kind
    "reference"; else the oracle port (oracle/cpu_session.py) -> kind "port"."""
    if (REF_DIR / "persistkern" / "native.py").exists():
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        from persistkern import native as ref_native
        from persistkern.device import WorkDescriptor as RefWork

        class _Ref:
            kind = "reference"
            name = "persistkern.native.NativeSession (baseline/_ref, unmodified)"

            def __init__(self, workers, threshold):
                self.s, _ = ref_native.NativeSession.start(
                    ref_native.NativeConfig(num_workers=workers, spin_yield_threshold=threshold))
                self.w = RefWork(slot=0, iterations=0)

            def roundtrip(self, m):
                self.s.trigger(m, self.w)
                self.s.wait(m)

            def close(self):
                self.s.dispose()
        return _Ref
    from oracle.cpu_session import CpuSession

    class _Port:
        kind = "port"
        name = "oracle/cpu_session.py (thread-per-worker port of persistkern.native)"

        def __init__(self, workers, threshold):
            self.s = CpuSession(num_workers=workers, spin_yield_threshold=threshold)
            self.s.start()

        def roundtrip(self, m):
            self.s.trigger(m, 0)
            self.s.wait(m)

        def close(self):
            self.s.dispose()
    return _Port


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's own CPU executor on our arm's config
    (148 workers, empty task, round-robin single-worker masks)."""
    if rank != 0:
        return
    workers = args.workers or 148
    threshold = 200   # the reference test suite's setting (T/test_native.py:13); 10k default is ~20x slower here
    Exe = reference_executor()
    t_init = time.perf_counter()
    s = Exe(workers, threshold)
    init_s = time.perf_counter() - t_init
    per_step = args.ref_rounds or max(1, -(-1000 // max(1, args.steps)))   # >= 1,000 timed round trips
    k = 0
    for _ in range(args.warmup):
        for kk in range(k, k + per_step):
            s.roundtrip(1 << (kk % workers))
        k += per_step
    lat = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for kk in range(k, k + per_step):
            a = time.perf_counter_ns()
            s.roundtrip(1 << (kk % workers))
            lat.append(time.perf_counter_ns() - a)
        k += per_step
    dt = time.perf_counter() - t0
    s.close()
    rounds = per_step * args.steps
    value = rounds / dt
    cores = len(os.sched_getaffinity(0))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "tasks/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * dt / args.steps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"configs[1] shape on the CPU executor: empty-task round-robin dispatch, "
                               f"{workers} persistent workers", "rounds_per_step": per_step,
                   "executor": Exe.name, "spin_yield_threshold": threshold,
                   "init_s": round(init_s, 3)},
        "latency_us": lat_summary(lat),
        "cpu_baseline": {"value": round(value, 3), "unit": "tasks/s", "cores": cores, "kind": Exe.kind,
                         "sample": f"{rounds} round trips on {workers} Python worker threads "
                                   f"(GIL-bound; {cores} host threads available)", "host": host_info()},
        "e2e": {"value": round(value, 3), "unit": "tasks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def thread_driver_rows(rows):
    """Aggregate per-GPU rows of the --threads run: whole-job tasks/s = all
    GPUs' rounds / the slowest GPU's time (the max-over-ranks rule)."""
    t = max(r["elapsed_s"] for r in rows)
    units = sum(r["rounds"] for r in rows)
    return units / t, t, units


def run_threads_arm(args):
    """configs[4] in the north star's form: ONE process, one LK session per
    visible GPU, each driven by its own host thread pinned to a core local to
    its GPU's NUMA node (P/native.py:70-79's pinning concept), all timed
    between two thread barriers.  Independent instances: no collective, no
    shared state but the barrier."""
    from paper_2310_01212_b200 import native
    from paper_2310_01212_b200.device import WorkDescriptor
    ndev = native.device_count()
    gpus = args.gpus if args.gpus and args.gpus <= ndev else ndev
    start_bar = threading.Barrier(gpus)
    end_bar = threading.Barrier(gpus)
    rows = [None] * gpus
    errs = []
    taken = set()
    lock = threading.Lock()

    def drive(d):
        try:
            native.init_device(d)
            native.pin_host_thread(d)
            local_cores = sorted(os.sched_getaffinity(0))
            with lock:   # one core per thread, highest-numbered free one of the GPU's set
                core = next((c for c in reversed(local_cores) if c not in taken), local_cores[-1])
                taken.add(core)
            os.sched_setaffinity(0, {core})
            cfg = native.NativeConfig(num_workers=args.workers, device=d, spin_strategy=native.PURE_SPIN)
            s, _ = native.NativeSession.start(cfg)
            try:
                s.register(WorkDescriptor(slot=0, kind="empty"))
                rr = [1 << i for i in range(s.num_workers)]
                for _ in range(args.warmup):
                    s.bench_roundtrip(rr, 0, args.rounds)
                start_bar.wait()
                t0 = time.perf_counter_ns()
                done = [s.bench_roundtrip(rr, 0, args.rounds)[1] for _ in range(args.steps)]
                el = (time.perf_counter_ns() - t0) / 1e9
                end_bar.wait()
                done = np.concatenate(done)
                rows[d] = {"device": d, "core": core, "workers": s.num_workers, "rounds": int(done.size),
                           "elapsed_s": el, "tasks_per_s": round(done.size / el, 1),
                           "trigger_to_done": lat_summary(done)}
                s.dispose()
            finally:
                s.close()
        except Exception as exc:   # report; abort the barriers so the other threads do not wait forever
            errs.append(f"gpu {d}: {exc!r}")
            start_bar.abort()
            end_bar.abort()

    ths = [threading.Thread(target=drive, args=(d,)) for d in range(gpus)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        print(json.dumps({"metric": METRIC, "error": errs}), flush=True)
        return
    value, t_max, units = thread_driver_rows(rows)
    line = {"metric": METRIC, "value": round(value, 1), "unit": "tasks/s", "n_gpus": gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * t_max / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "configs[4]: independent LK instances, one per GPU, one NUMA-pinned host "
                                   "thread each, in one process (configs[1] loop on every GPU)",
                       "parallelism": f"threads{gpus}", "rounds_per_step": args.rounds},
            "gpu_launches": gpus, "per_gpu": rows}
    print(json.dumps(line), flush=True)


METRIC = "trigger->done round trips per second (empty task, 148 persistent workers)"
# extras printed at the end of the JSON line, next to the latency headline
HEADLINE_EXTRAS = ("single_worker", "full_mask", "full_mask_payload_session", "interference", "interference_green",
                   "pingpong_floor",
                   "tail_attribution")


# ----------------------------------------------------------------------------- LK arm

def measure_payload(session, kind, sizes_mib, reps, rotate_bytes):
    """GB/s of a payload kind dispatched to all workers, L2-cold by rotation."""
    from paper_2310_01212_b200 import host
    from paper_2310_01212_b200.device import BYTES_PER_ELEMENT, DeviceBuffer, WorkDescriptor, reduce_blocks
    full = host.full_mask(session.num_workers)
    out = {}
    for mib in sizes_mib:
        n = (mib << 20) // 4
        per_set = (8 if kind == "saxpy_f32" else 4) * n
        sets = max(2, min(64, -(-rotate_bytes // per_set)))
        bufs, works = [], []
        for k in range(sets):
            if kind == "saxpy_f32":
                x, y = DeviceBuffer(4 * n), DeviceBuffer(4 * n)
                bufs += [x, y]
                works.append(WorkDescriptor(slot=100 + k, kind=kind, data_in_ref=(x, y), data_out_ref=y, alpha=1.5))
            else:
                x, p, t = DeviceBuffer(4 * n), DeviceBuffer(8 * reduce_blocks(n)), DeviceBuffer(8)
                bufs += [x, p, t]
                works.append(WorkDescriptor(slot=100 + k, kind=kind, data_in_ref=x, data_out_ref=p, total_ref=t))
        for w in works:
            session.register(w, full)
        spans, e2e = [], []
        for r in range(reps + 2):
            w = works[r % sets]
            t0 = time.perf_counter_ns()
            session.trigger(full, w)
            session.wait(full)
            t1 = time.perf_counter_ns()
            b, e = session.last_spans()
            if r >= 2:
                spans.append(int(e.max()) - int(b.min()))
                e2e.append(t1 - t0)
        nbytes = BYTES_PER_ELEMENT[kind] * n
        med_span = statistics.median(spans)
        out[f"{mib}MiB"] = {"bytes": nbytes, "device_span_us": round(med_span / 1e3, 3),
                            "gbs_device": round(nbytes / med_span, 1),
                            "gbs_e2e": round(nbytes / statistics.median(e2e), 1),
                            "rotation_sets": sets}
        for bf in bufs:
            bf.free()
    return out


def measure_config0(session, rounds, n=65536):
    from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor
    a = np.random.default_rng(0).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    b = np.random.default_rng(1).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    da, db = DeviceBuffer.from_array(a), DeviceBuffer.from_array(b)
    outs = [DeviceBuffer(4 * n) for _ in range(4)]
    works = [WorkDescriptor(slot=700 + i, kind="vector_add_i32", data_in_ref=(da, db), data_out_ref=outs[i])
             for i in range(4)]
    for i, w in enumerate(works):
        session.register(w, 1 << i)
    for k in range(200):
        session.trigger(1 << (k % 4), works[k % 4])
        session.wait(1 << (k % 4))
    lat = []
    t0 = time.perf_counter_ns()
    for k in range(rounds):
        m = 1 << (k % 4)
        a0 = time.perf_counter_ns()
        session.trigger(m, works[k % 4])
        session.wait(m)
        lat.append(time.perf_counter_ns() - a0)
    dt = (time.perf_counter_ns() - t0) / 1e9
    for buf in [da, db] + outs:
        buf.free()
    return {"what": "configs[0] workload on the GPU: 4 workers round robin, one int32 vector add of "
                    "64 Ki elements per task, Python API trigger+wait", "tasks_per_s": round(rounds / dt, 1),
            "latency": lat_summary(lat),
            "parity": "tests/test_gpu_payload.py::test_vector_add_i32_bit_exact (same kind, sizes, masks)"}


_LOCAL_CORES: list = []
_ALLOWED_CORES: list = []   # the process's affinity before the LK arm pinned its host thread


def host_info():
    """The CPU side of the comparison: what the reference
    executor's Python threads ran on."""
    import platform
    return {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "python": platform.python_version(), "switchinterval_s": sys.getswitchinterval(),
            "cpu": platform.processor() or platform.machine()}


def read_only_peak(device):
    try:
        import torch
        x = torch.empty(1 << 28, dtype=torch.float32, device=f"cuda:{device}").uniform_()
        for _ in range(3):
            x.sum()
        best = None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(10):
            e0.record()
            x.sum()
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del x
        return round((1 << 30) / (best * 1e6), 1)
    except Exception:
        return None


def measure_interference_green(cfg, lat_sms, rounds, stream_mib):
    """configs[3] with a hardware partition: the LK session runs in a green
    context of lat_sms SMs (16); an ordinary hbm_stream kernel (the baseline's
    work kernel, same TMA copy code) runs back to back on the remaining SMs'
    green context from a second host thread on its own core."""
    from paper_2310_01212_b200 import native
    from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor
    gs, _ = native.NativeSession.start(dataclasses.replace(cfg, sm_partition=lat_sms, num_workers=None))
    masks = [1 << i for i in range(gs.num_workers)]
    gs.register(WorkDescriptor(slot=0, kind="empty"))
    gs.bench_roundtrip(masks, 0, 5000)
    _, solo, _ = gs.bench_roundtrip(masks, 0, rounds)
    b = native.LaunchSyncBaseline(beside=gs)
    elems = (stream_mib << 20) // 4
    src, dst = DeviceBuffer(4 * elems), DeviceBuffer(4 * elems)
    sw = WorkDescriptor(slot=0, kind="hbm_stream", data_in_ref=src, data_out_ref=dst, iterations=1)
    b.time_kernel(sw, 1)
    stop = threading.Event()
    gbs = []
    mine = sorted(os.sched_getaffinity(0))
    others = [c for c in sorted(_LOCAL_CORES or mine) if c not in mine] or mine

    def streamer():
        try:
            os.sched_setaffinity(0, {others[-1]})
        except OSError:
            pass
        while not stop.is_set():
            ms = b.time_kernel(sw, 4)            # average ms per launch
            gbs.append(8 * elems / (ms * 1e6))

    th = threading.Thread(target=streamer, daemon=True)
    th.start()
    while len(gbs) < 2:
        time.sleep(0.001)
    _, co, _ = gs.bench_roundtrip(masks, 0, rounds)
    stop.set()
    th.join()
    b.close()
    src.free()
    dst.free()
    lk_sms, rest = gs.partition_info
    gs.dispose()
    gs.close()
    return {"latency_partition_sms": lk_sms, "stream_partition_sms": rest,
            "solo": lat_summary(solo), "co_running": lat_summary(co),
            "jitter_delta_us": round((pct(co, 99.9) - pct(co, 50)) / 1e3 - (pct(solo, 99.9) - pct(solo, 50)) / 1e3, 3),
            "stream_gbs_cuda_events": round(statistics.median(gbs), 1), "stream_batches": len(gbs),
            "note": "green-context SM partitions (cuGreenCtxCreate); the stream partition runs ordinary "
                    "kernel launches (cudaLaunchKernel + events), not LK workers"}


def measure_lazy(cfg, masks, rounds):
    from paper_2310_01212_b200 import native
    from paper_2310_01212_b200.device import WorkDescriptor
    ls, _ = native.NativeSession.start(dataclasses.replace(cfg, lazy_ack=True))
    ls.register(WorkDescriptor(slot=0, kind="empty"))
    ls.bench_roundtrip(masks, 0, 5000)
    _, done, cyc = ls.bench_roundtrip(masks, 0, rounds)
    ls.dispose()
    ls.close()
    return {"tasks_per_s": round(rounds / (cyc.sum() / 1e9), 1), "trigger_to_done": lat_summary(done),
            "round_trip": lat_summary(cyc),
            "note": "NativeConfig(lazy_ack=True): the NOP ack's consumption is awaited by the worker's "
                    "next trigger instead of inside wait(); protocol and traces unchanged"}


def measure_table2(device, reps=100, iterations=20_000):
    """The paper's Table II scenarios (P/bench.py:358-373: table2-single-sm,
    table2-full-gpu; busy_loop work of 20,000 iterations, 100 reps) on B200
    hardware through backend.run_b200: LK Init/Trigger/Wait/Dispose vs the
    launch+sync baseline's Alloc/Launch/Wait/Dispose, in ns (avg / worst)."""
    from paper_2310_01212_b200 import backend, host
    from paper_2310_01212_b200.device import WorkDescriptor

    class Scn:
        def __init__(self, scope, n):
            self.reps, self.scope, self.n = reps, scope, n

        def cluster_count(self):
            return self.n

        def mask(self):
            return 1 if self.scope == "single_sm" else host.full_mask(self.n)

        def work(self):
            return WorkDescriptor(slot=0, iterations=iterations)

        def models(self):
            return [host.MODEL_LK, host.MODEL_BASELINE]

    from paper_2310_01212_b200 import _lib
    import ctypes as C
    nsm = C.c_int()
    _lib.check(_lib.load().lk_sm_count(device, C.byref(nsm)))
    out = {}
    for scope in ("single_sm", "full_gpu"):
        rows = backend.run_b200(Scn(scope, nsm.value), device=device)
        out[f"table2-{scope.replace('_', '-')}"] = {f"{r.model}/{r.phase}": {"avg_ns": round(r.avg, 1),
                                                                           "worst_ns": r.worst}
                                                   for r in rows}
    return out


def measure_small_transfer(device, reps):
    from paper_2310_01212_b200.device import DeviceBuffer
    buf = DeviceBuffer(4096, device)
    h = np.zeros(1, dtype=np.uint32)
    up, down = [], []
    for k in range(reps + 100):
        h[0] = k
        t0 = time.perf_counter_ns()
        buf.upload(h)
        t1 = time.perf_counter_ns()
        h[:] = buf.download(np.uint32, 1)
        t2 = time.perf_counter_ns()
        if k >= 100:
            up.append(t1 - t0)
            down.append(t2 - t1)
    buf.free()
    return {"h2d_4B_memcpy": lat_summary(up), "d2h_4B_memcpy": lat_summary(down),
            "note": "cudaMemcpyAsync + stream sync of 4 bytes through the Python API (DeviceBuffer "
                    "upload/download); compare the mailbox word round trip in latency_us"}


def measure_zero_copy(cfg, device, sizes, reps):
    """The paper's small-transfer case on B200 (P/link.py:
    84-122; P/host.py:212-224): one int32 vector add of `b` bytes per input
    on ONE worker, inputs from the host and the result back to the host, per
    task, end to end:
      lk_zero_copy   HostBuffer in/out (LK_DF_HOSTMEM), trigger+wait only
                     (closed loop in C: lk_bench_roundtrip)
      lk_copies      DeviceBuffers: 2 cudaMemcpy H2D + trigger+wait + 1 D2H
      launch_copies  the conventional flow: 2 H2D + launch + sync + D2H
      launch_zero_copy  launch + sync with the HostBuffers
    Then the mailbox-only single-worker sync against the paper's full-board
    workaround (LK_CF_FULL_BOARD: every write re-ships all 148 cells)."""
    from paper_2310_01212_b200 import native
    from paper_2310_01212_b200.device import DeviceBuffer, HostBuffer, WorkDescriptor
    rng = np.random.default_rng(0)
    bufs = {}
    for b in sizes:
        n = max(1, b // 4)
        a = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
        c = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
        bufs[b] = (n, a, c, HostBuffer.from_array(a, device), HostBuffer.from_array(c, device),
                   HostBuffer(4 * n, device), DeviceBuffer(4 * n, device), DeviceBuffer(4 * n, device),
                   DeviceBuffer(4 * n, device))
    out = {"sizes_bytes": list(sizes), "reps": reps}
    zcfg = dataclasses.replace(cfg, poll_mode="direct", full_board=False)
    s, _ = native.NativeSession.start(zcfg)
    rows = {}
    ok = True
    for k, b in enumerate(sizes):
        n, a, c, ha, hc, ho, da, dc, do = bufs[b]
        zw = WorkDescriptor(slot=700 + k, kind="vector_add_i32", data_in_ref=(ha, hc), data_out_ref=ho)
        s.register(zw, 1)
        s.bench_roundtrip([1], 700 + k, 200)
        _, zdone, zcyc = s.bench_roundtrip([1], 700 + k, reps)
        ok &= bool(np.array_equal(ho.array(np.int32, n), a + c))
        cw = WorkDescriptor(slot=720 + k, kind="vector_add_i32", data_in_ref=(da, dc), data_out_ref=do)
        res = np.empty(n, np.int32)
        lat = []
        for r in range(reps // 4 + 50):
            t0 = time.perf_counter_ns()
            da.upload(a)
            dc.upload(c)
            s.trigger(1, cw)
            s.wait(1)
            res[:] = do.download(np.int32, n)
            if r >= 50:
                lat.append(time.perf_counter_ns() - t0)
        ok &= bool(np.array_equal(res, a + c))
        s.timings.clear()
        rows[b] = {"lk_zero_copy": lat_summary(zcyc), "lk_zero_copy_trigger_to_done": lat_summary(zdone),
                   "lk_copies": lat_summary(lat)}
    s.dispose()
    s.close()
    base = native.LaunchSyncBaseline(device=device, grid=1)
    for k, b in enumerate(sizes):
        n, a, c, ha, hc, ho, da, dc, do = bufs[b]
        cw = WorkDescriptor(slot=0, kind="vector_add_i32", data_in_ref=(da, dc), data_out_ref=do)
        zw = WorkDescriptor(slot=0, kind="vector_add_i32", data_in_ref=(ha, hc), data_out_ref=ho)
        lat, zl = [], []
        res = np.empty(n, np.int32)
        for r in range(reps // 4 + 50):
            t0 = time.perf_counter_ns()
            da.upload(a)
            dc.upload(c)
            base.launch(cw, 1)
            base.wait()
            res[:] = do.download(np.int32, n)
            t1 = time.perf_counter_ns()
            base.launch(zw, 1)
            base.wait()
            t2 = time.perf_counter_ns()
            if r >= 50:
                lat.append(t1 - t0)
                zl.append(t2 - t1)
        ok &= bool(np.array_equal(res, a + c)) and bool(np.array_equal(ho.array(np.int32, n), a + c))
        rows[b]["launch_copies"] = lat_summary(lat)
        rows[b]["launch_zero_copy"] = lat_summary(zl)
    base.close()
    out["per_size"] = rows
    out["results_exact"] = ok
    # mailbox bytes only vs the full board, single-worker round robin over every worker
    board = {}
    for name, fb in (("mailbox_word", False), ("full_board", True)):
        bs, _ = native.NativeSession.start(dataclasses.replace(cfg, poll_mode="direct", full_board=fb))
        bs.register(WorkDescriptor(slot=0, kind="empty"))
        m = [1 << i for i in range(bs.num_workers)]
        bs.bench_roundtrip(m, 0, 2000)
        _, d, cy = bs.bench_roundtrip(m, 0, reps)
        board[name] = {"trigger_to_done": lat_summary(d), "round_trip": lat_summary(cy)}
        bs.dispose()
        bs.close()
    board["note"] = ("the paper had to ship the whole mailbox board for a single-SM trigger because the "
                     "driver deferred tiny transfers (PAPER.md:157-160); mapped sys-scope stores are never "
                     "deferred, so the single 8-B word completes and the board costs only extra stores")
    out["single_sm_sync"] = board
    out["note"] = ("per task, host->device inputs and device->host result included; lk_zero_copy from C "
                   "(lk_bench_roundtrip), the copy flows through the Python API (DeviceBuffer.upload/"
                   "download: cudaMemcpyAsync + stream sync)")
    return out


def measure_multi_driver(session, drivers, rounds):
    n = session.num_workers
    groups = [list(range(g, n, drivers)) for g in range(drivers)]
    res = [None] * drivers
    mine = sorted(os.sched_getaffinity(0))
    cores = [c for c in sorted(_LOCAL_CORES or mine) if c not in mine] or mine

    from paper_2310_01212_b200.device import WorkDescriptor
    for g in range(drivers):   # one slot per driver: a slot is locked while un-waited (native.py:215-217)
        session.register(WorkDescriptor(slot=800 + g, kind="empty"))

    def drive(g):
        try:
            os.sched_setaffinity(0, {cores[g % len(cores)]})
        except OSError:
            pass
        _, done, cyc = session.bench_roundtrip([1 << i for i in groups[g]], 800 + g, rounds)
        res[g] = (done, cyc)

    ths = [threading.Thread(target=drive, args=(g,)) for g in range(drivers)]
    t0 = time.perf_counter_ns()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = (time.perf_counter_ns() - t0) / 1e9
    done = np.concatenate([r[0] for r in res])
    return {"drivers": drivers, "workers_per_driver": len(groups[0]), "rounds_per_driver": rounds,
            "aggregate_tasks_per_s": round(drivers * rounds / dt, 1), "trigger_to_done": lat_summary(done),
            "note": "each host thread on its own GPU-local core runs lk_bench_roundtrip over a disjoint "
                    "worker group (round robin) of one session"}


def measure_interference(session, lat_workers, rounds, stream_mib):
    """configs[3]: a latency partition (workers [0, lat_workers), closed-loop
    empty tasks round-robin, driven from C) measured solo, then while the
    other workers run hbm_stream (src -> dst, stream_mib MiB each) re-triggered
    back to back by a second host thread.  Same session, disjoint worker sets,
    so the two host threads never contend for a worker."""
    from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor
    n = session.num_workers
    lat_masks = [1 << i for i in range(lat_workers)]
    stream_mask = ((1 << n) - 1) & ~((1 << lat_workers) - 1)
    elems = (stream_mib << 20) // 4
    src, dst = DeviceBuffer(4 * elems), DeviceBuffer(4 * elems)
    sw = WorkDescriptor(slot=900, kind="hbm_stream", data_in_ref=src, data_out_ref=dst, iterations=1)
    session.register(sw, stream_mask)
    session.register(WorkDescriptor(slot=0, kind="empty"))
    session.bench_roundtrip(lat_masks, 0, 5000)
    _, solo, _ = session.bench_roundtrip(lat_masks, 0, rounds)

    stop = threading.Event()
    stream_stats = {"dispatches": 0, "ns": 0, "spans_ns": []}

    # the streaming partition's host thread gets its own core: threads inherit
    # the creator's affinity, and two spinning threads on one core would turn
    # the latency partition's tail into scheduler time slices
    mine = sorted(os.sched_getaffinity(0))
    local = sorted(_LOCAL_CORES or mine)
    others = [c for c in local if c not in mine] or [c for c in range(os.cpu_count() or 1) if c not in mine]

    def streamer():
        if others:
            try:
                os.sched_setaffinity(0, {others[-1]})
            except OSError:
                pass
        t0 = time.perf_counter_ns()
        while not stop.is_set():
            session.trigger(stream_mask, sw)
            session.wait(stream_mask)
            stream_stats["dispatches"] += 1
        stream_stats["ns"] = time.perf_counter_ns() - t0

    th = threading.Thread(target=streamer, daemon=True)
    th.start()
    while stream_stats["dispatches"] < 2:
        time.sleep(0.001)
    _, co, _ = session.bench_roundtrip(lat_masks, 0, rounds)
    stop.set()
    th.join()
    b, e = session.last_spans()
    span = int(e[lat_workers:].max()) - int(b[lat_workers:].min())
    src.free()
    dst.free()
    moved = 8 * elems * stream_stats["dispatches"]
    return {"latency_partition_workers": lat_workers, "stream_partition_workers": n - lat_workers,
            "stream_bytes_per_dispatch": 8 * elems,
            "solo": lat_summary(solo), "co_running": lat_summary(co),
            "jitter_delta_us": round((pct(co, 99.9) - pct(co, 50)) / 1e3 - (pct(solo, 99.9) - pct(solo, 50)) / 1e3, 3),
            "stream_gbs_host": round(moved / max(1, stream_stats["ns"]), 1),
            "stream_gbs_device_last": round(8 * elems / max(1, span), 1),
            "stream_dispatches": stream_stats["dispatches"]}


def standalone_kernel_gbs(device, kind, mib, reps=20):
    """Same work function as an ordinary kernel (148 CTAs), CUDA-event timed."""
    from paper_2310_01212_b200 import native
    from paper_2310_01212_b200.device import BYTES_PER_ELEMENT, DeviceBuffer, WorkDescriptor
    n = (mib << 20) // 4
    sets = 6
    b = native.LaunchSyncBaseline(device=device)
    bufs, works = [], []
    for k in range(sets):
        x, y = DeviceBuffer(4 * n, device), DeviceBuffer(4 * n, device)
        bufs += [x, y]
        works.append(WorkDescriptor(slot=0, kind=kind, data_in_ref=(x, y), data_out_ref=y, alpha=1.5))
    ms = []
    for r in range(reps):
        ms.append(b.time_kernel(works[r % sets], 1))
    b.close()
    for bf in bufs:
        bf.free()
    med = statistics.median(ms[2:])
    return {"ms": round(med, 4), "gbs": round(BYTES_PER_ELEMENT[kind] * n / (med * 1e6), 1)}


def run_lk_arm(args, world, rank, local):
    from paper_2310_01212_b200 import host, native
    from paper_2310_01212_b200.device import WorkDescriptor

    device = local
    pinned = 0
    pinned_core = None
    _ALLOWED_CORES[:] = sorted(os.sched_getaffinity(0))
    # bring the CUDA context (and the driver's helper threads) up before the
    # host thread is pinned: threads inherit their creator's affinity, and a
    # driver thread sharing the pinned core would preempt the spin loop
    native.init_device(device)
    try:
        pinned = native.pin_host_thread(device)
        # one core of the GPU-local set, the highest-numbered one (core 0 takes
        # most housekeeping interrupts): no migrations under the spin loop
        local_cores = sorted(os.sched_getaffinity(0))
        _LOCAL_CORES[:] = local_cores
        pinned_core = local_cores[-1 - (local % max(1, len(local_cores)))]
        os.sched_setaffinity(0, {pinned_core})
    except Exception:
        pinned = 0
    # under ncu (which serialises launches) the same command still runs: the
    # descriptors live in mapped host memory and the legs that make CUDA
    # calls while a session is resident (payload buffers, cudaMemcpy probes,
    # the payload/interference/zero-copy sessions) are skipped. The line is
    # then a launch-list run, not a bench value.
    prof = native.under_profiler()
    if prof:
        args.no_payload = args.no_interference = args.no_lazy = args.no_green = True
        args.no_zero_copy = args.no_table2 = True
    cfg = native.NativeConfig(num_workers=args.workers, device=device, spin_strategy=native.PURE_SPIN,
                              poll_backoff_ns=args.backoff_ns, cell_stride=args.cell_stride,
                              poll_replicas=args.replicas, poll_spacing_ns=args.spacing_ns,
                              poll_mode=args.poll_mode, tma_payload=not args.lsu_payload,
                              host_descriptors=prof)
    session, init = native.NativeSession.start(cfg)
    n = session.num_workers
    empty = WorkDescriptor(slot=0, kind="empty")
    session.register(empty)
    rr_masks = [1 << i for i in range(n)]
    R = args.rounds

    for _ in range(args.warmup):
        session.bench_roundtrip(rr_masks, 0, R)

    barrier(world)
    done_all, cyc_all = [], []
    with ClockSampler(device, pinned_core) as clk, CoreNoise(pinned_core if pinned_core is not None else 0) as noise:
        t0 = time.perf_counter_ns()
        for _ in range(args.steps):
            _, done, cyc = session.bench_roundtrip(rr_masks, 0, R)
            done_all.append(done)
            cyc_all.append(cyc)
        t1 = time.perf_counter_ns()
    barrier(world)
    elapsed = (t1 - t0) / 1e9
    rounds = R * args.steps
    t_max, units = gather_max_sum(world, elapsed, rounds)
    value = units / t_max
    done_all = np.concatenate(done_all)
    cyc_all = np.concatenate(cyc_all)
    # configs[4]: every GPU's own p50/p99.9 beside the aggregate (rank = GPU)
    mine = lat_summary(done_all)
    per_rank = gather_rank_rows(world, {"rank": rank, "device": device, "rounds": int(done_all.size),
                                        "elapsed_s": round(elapsed, 6), "tasks_per_s": round(rounds / elapsed, 1),
                                        "p50_us": mine["p50_us"], "p99.9_us": mine["p99.9_us"]})

    extras = {}
    if not prof:   # a device->host copy of the timeline words
        tl = session.last_timeline().astype(np.int64)
        dev_cyc = (tl[:, 7] - tl[:, 5]).astype(np.float64)
        extras["device_handling"] = {
            "what": "clock64 cycles, each worker's last timed dispatch: to_gpu value seen -> FINISHED store issued",
            "p50_cycles": float(np.median(dev_cyc)), "max_cycles": float(dev_cyc.max()),
            "p50_us_at_max_clock": round(float(np.median(dev_cyc)) / SM_MAX_GHZ / 1e3, 4)}
    # tail attribution (untimed): the same loop with the host thread's own
    # spin gaps recorded per round; a round slower than p50 + 2 us whose host
    # thread stalled >= 1 us was slowed on the host side, not on the link/GPU
    with CoreNoise(pinned_core if pinned_core is not None else 0) as anoise:
        _, adone, _, agap = session.bench_roundtrip_gaps(rr_masks, 0, args.attrib_rounds)
    a50 = float(np.percentile(adone, 50))
    slow = adone > a50 + 2000
    stalled = agap >= 1000
    clean = adone[~stalled]
    extras["tail_attribution"] = {
        "rounds": int(adone.size), "trigger_to_done": lat_summary(adone),
        "slow_rounds": int(slow.sum()), "slow_rounds_with_host_stall_ge_1us": int((slow & stalled).sum()),
        "rounds_with_host_stall_ge_1us": int(stalled.sum()),
        "host_stall_us": lat_summary(agap[stalled]) if stalled.any() else None,
        "trigger_to_done_without_host_stall": lat_summary(clean) if clean.size else None,
        "host_noise": anoise.summary(),
        "note": "host stall = largest gap between consecutive TSC reads of the pinned host thread inside "
                "the round (lk_bench_roundtrip_gaps); the rounds without one show the link+GPU alone"}
    # full-148-worker dispatch
    full = host.full_mask(n)
    _, fdone, fcyc = session.bench_roundtrip([full], 0, args.full_rounds)
    extras["full_mask"] = {"trigger_to_done": lat_summary(fdone), "round_trip": lat_summary(fcyc),
                           "tasks_per_s": round(args.full_rounds / (fcyc.sum() / 1e9), 1)}
    # one worker re-triggered back to back (the adaptive idle delay's case),
    # from C and through the Python API
    _, sdone, scyc = session.bench_roundtrip([1], 0, 3000)
    _, sdone, scyc = session.bench_roundtrip([1], 0, args.full_rounds)
    empty_w = WorkDescriptor(slot=0, kind="empty")
    for _k in range(2000):
        session.trigger(1, empty_w)
        session.wait(1)
    t_py = time.perf_counter_ns()
    for _k in range(args.full_rounds):
        session.trigger(1, empty_w)
        session.wait(1)
    t_py = time.perf_counter_ns() - t_py
    session.timings.clear()
    extras["single_worker"] = {"trigger_to_done": lat_summary(sdone), "round_trip": lat_summary(scyc),
                               "tasks_per_s": round(args.full_rounds / (scyc.sum() / 1e9), 1),
                               "python_api_tasks_per_s": round(args.full_rounds / (t_py / 1e9), 1),
                               "note": "worker 0 re-triggered back to back (adaptive idle delay engaged)"}

    # the small-transfer case the paper's pathology is about (PAPER:160-162,
    # P/link.py:84-122): a 4-byte cudaMemcpy each way (stream-synchronous)
    # next to the mailbox word round trip above
    if rank == 0 and not prof:
        extras["small_transfer"] = measure_small_transfer(device, 2000)

    # several host threads, each a closed loop over its own worker group (one
    # session; disjoint workers): aggregate tasks/s a B200 sustains
    if rank == 0 and args.drivers > 1:
        extras["multi_driver"] = measure_multi_driver(session, args.drivers, args.driver_rounds)

    # e2e through the Python API (reference-facing plugin), host buffers = mailbox words
    e2e_rounds = args.e2e_rounds
    barrier(world)
    t0 = time.perf_counter_ns()
    for k in range(e2e_rounds):
        m = rr_masks[k % n]
        session.trigger(m, empty)
        session.wait(m)
    e2e_dt = (time.perf_counter_ns() - t0) / 1e9
    barrier(world)
    e2e_t, e2e_units = gather_max_sum(world, e2e_dt, e2e_rounds)
    e2e_value = e2e_units / e2e_t          # whole job: all ranks' tasks / slowest rank

    # 64 MiB saxpy on this DIRECT session too: its per-worker early acks make
    # the wide handshake cheaper end to end, the gateway's single ring event
    # makes the start skew (and so the device span) smaller
    if rank == 0 and not args.no_payload:
        extras["payload_direct"] = {"saxpy_f32": measure_payload(session, "saxpy_f32", [64], args.payload_reps,
                                                                 4 * L2_BYTES),
                                    "poll_mode": "direct"}

    # configs[0] shape on the GPU: 4 workers round robin, int32 vector add of 64 Ki
    # elements per task (the CPU reference's workload), trigger->done per task
    if rank == 0 and not args.no_payload:
        extras["config0_on_gpu"] = measure_config0(session, args.config0_rounds)

    smids = session.smid_map
    session.dispose()
    session.close()

    if rank == 0 and not args.no_interference and not args.no_green:
        try:
            extras["interference_green"] = measure_interference_green(cfg, args.lat_workers,
                                                                      args.interf_rounds, args.stream_mib)
        except Exception as exc:   # green contexts need driver support; report, don't fail the bench
            extras["interference_green"] = {"error": str(exc)}

    # lazy ack (opt-in): wait() returns once the ack is written; the round
    # robin's next worker is another one, so the ack's consumption overlaps.
    # (Each extra session starts after the previous one is disposed: a live
    # session owns every SM.)
    if rank == 0 and not args.no_lazy:
        extras["lazy_ack"] = measure_lazy(cfg, rr_masks, args.lazy_rounds)

    # configs[2]: payload items dispatched to every worker, on a HYBRID
    # session: the trigger is one ring event (it reaches all 148 workers
    # within ~0.5 us; direct polling spreads their start over ~2 us, which the
    # span -- and so the GB/s -- would include at small sizes), and the acks
    # go to the direct cells as each FINISHED is seen.
    payload = {}
    if not args.no_payload and rank == 0:
        pcfg = dataclasses.replace(cfg, poll_mode=args.payload_poll_mode)
        psession, _ = native.NativeSession.start(pcfg)
        payload["poll_mode"] = args.payload_poll_mode
        payload["saxpy_f32"] = measure_payload(psession, "saxpy_f32", args.payload_mib, args.payload_reps,
                                               4 * L2_BYTES)
        payload["block_reduce_f32"] = measure_payload(psession, "block_reduce_f32", args.payload_mib,
                                                      args.payload_reps, 4 * L2_BYTES)
        # steady state: at 64 MiB a worker streams ~28 tiles, so pipeline
        # fill, dispatch skew and the combine (~5 us together) are a third of
        # the reduce's span; at 1 GiB they vanish
        payload["block_reduce_f32_steady"] = measure_payload(psession, "block_reduce_f32", [1024], 6,
                                                             2 * L2_BYTES)
        # the empty full-mask dispatch on this session (triggers as one ring
        # event), beside the DIRECT session's full_mask above
        psession.register(WorkDescriptor(slot=0, kind="empty"))
        pfull = host.full_mask(psession.num_workers)
        psession.bench_roundtrip([pfull], 0, 2000)
        _, gdone, gcyc = psession.bench_roundtrip([pfull], 0, args.full_rounds)
        extras["full_mask_payload_session"] = {"poll_mode": args.payload_poll_mode,
                                               "trigger_to_done": lat_summary(gdone), "round_trip": lat_summary(gcyc),
                                               "tasks_per_s": round(args.full_rounds / (gcyc.sum() / 1e9), 1)}
        psession.dispose()
        psession.close()

    # configs[3]: latency partition beside an HBM-streaming partition, on a
    # HYBRID session: the latency workers' single-worker writes use their
    # direct cells, the 132-worker stream triggers travel as one ring event
    # each (one host store instead of 132, and no extra PCIe polling).
    if not args.no_interference and rank == 0 and n >= args.lat_workers + 8:
        icfg = dataclasses.replace(cfg, poll_mode=args.interference_poll_mode)
        isession, _ = native.NativeSession.start(icfg)
        extras["interference"] = measure_interference(isession, args.lat_workers, args.interf_rounds,
                                                      args.stream_mib)
        extras["interference"]["poll_mode"] = args.interference_poll_mode
        isession.dispose()
        isession.close()

    # zero-copy payloads vs cudaMemcpy for small transfers, and the full-board
    # mailbox workaround
    if rank == 0 and not args.no_zero_copy:
        try:
            extras["zero_copy"] = measure_zero_copy(cfg, device, [4, 64, 1024, 4096, 16384, 65536],
                                                    args.zc_reps)
        except Exception as exc:
            extras["zero_copy"] = {"error": repr(exc)}

    # conventional launch+sync baseline, same host thread
    base = {}
    b1 = native.LaunchSyncBaseline(device=device)
    for name, grid in (("grid1", 1), ("grid148", n)):
        b1.bench(empty, 200, grid)
        launch, total = b1.bench(empty, args.base_rounds, grid)
        base[name] = {"launch": lat_summary(launch), "launch_plus_sync": lat_summary(total)}
    # the same conventional flow through the Python API (launch() + wait() per
    # task), the counterpart of the LK arm's e2e
    n_py = min(args.e2e_rounds, 50_000)
    for _ in range(200):
        b1.launch(empty, 1)
        b1.wait()
    t0 = time.perf_counter_ns()
    for _ in range(n_py):
        b1.launch(empty, 1)
        b1.wait()
    base["python_api_tasks_per_s"] = round(n_py / ((time.perf_counter_ns() - t0) / 1e9), 1)
    b1.close()
    # the cheapest conventional flows (lk_launch_floor_bench): an empty
    # <<<1,32,0>>> kernel joined by stream sync, by a cudaStreamQuery spin,
    # or as a one-node graph; then the sync flow again under
    # cudaDeviceScheduleSpin (process-wide, so last)
    floor = {}
    for name, mode, spin in (("empty_kernel_sync", "kernel_sync", False), ("empty_kernel_query", "kernel_query", False),
                             ("graph_sync", "graph_sync", False), ("empty_kernel_sync_spinsched", "kernel_sync", True)):
        try:
            native.launch_floor(device, mode, 500, spin_sched=spin)
            tot, lau = native.launch_floor(device, mode, args.base_rounds, spin_sched=spin)
            floor[name] = {"launch_plus_sync": lat_summary(tot), "launch": lat_summary(lau)}
        except Exception as exc:  # pragma: no cover
            floor[name] = {"error": str(exc)}
    base["floor"] = floor
    if not prof:   # the ping-pong kernel waits on the host: a serialised launch would never return
        pp = native.pingpong(device, args.pp_rounds)
        extras["pingpong_floor"] = lat_summary(pp[100:])

    if rank != 0:
        return
    peak, peak_src = hbm_peak()
    roof = None
    if payload:
        big = f"{max(args.payload_mib)}MiB"
        ach = payload["saxpy_f32"][big]["gbs_device"]
        traffic = None
        tf = ROOT / "profiles" / "saxpy_traffic.json"
        if tf.exists():
            try:
                traffic = json.loads(tf.read_text()).get("bytes_per_launch")
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "kernel": f"lk_persistent_kernel saxpy_f32 {big} (148 workers)",
                "achieved": ach, "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes": payload["saxpy_f32"][big]["bytes"],
                "timing": "device %globaltimer span, first worker begin -> last worker end"}
        try:
            extras["standalone_saxpy_kernel"] = standalone_kernel_gbs(device, "saxpy_f32", max(args.payload_mib))
        except Exception as exc:  # pragma: no cover
            extras["standalone_saxpy_kernel"] = {"error": str(exc)}
        # the reduction reads only.  Its peak is the measured copy figure like
        # saxpy's; a read-only stream can exceed it (no read/write turnaround),
        # and torch.sum over 1 GiB is reported beside it for scale
        if "block_reduce_f32" in payload:
            rach = payload["block_reduce_f32"][big]["gbs_device"]
            steady = payload.get("block_reduce_f32_steady", {}).get("1024MiB", {}).get("gbs_device")
            extras["reduce_roofline"] = {"bound": "hbm (read-only)", "achieved": rach, "peak": peak,
                                         "unit": "GB/s", "frac": round(rach / peak, 4), "peak_source": peak_src,
                                         "achieved_1GiB": steady,
                                         "frac_1GiB": round(steady / peak, 4) if steady else None,
                                         "torch_sum_1GiB_gbs": read_only_peak(device),
                                         "kernel": f"lk_persistent_kernel block_reduce_f32 {big}"}

    if rank == 0 and not args.no_table2:
        extras["table2_b200"] = measure_table2(device)

    cpu = None
    if not args.no_cpu_baseline:
        # the reference's threads get the process's whole CPU set back: the LK
        # arm pinned this thread to one core, and threads inherit affinity
        try:
            os.sched_setaffinity(0, set(_ALLOWED_CORES) or os.sched_getaffinity(0))
        except OSError:
            pass
        cores = len(os.sched_getaffinity(0))
        cv, clat, ckind = cpu_baseline_config0(budget_s=0.6 * args.cpu_budget_s)
        cv2, clat2, _ = cpu_baseline_config0(threshold=200, budget_s=0.25 * args.cpu_budget_s)
        spawn = cpu_spawn_baseline_config0(budget_s=0.15 * args.cpu_budget_s)
        cpu = {"value": round(cv, 2), "unit": "tasks/s", "cores": cores, "kind": ckind, "host": host_info(),
               "sample": f"{len(clat)} round trips of BASELINE config 0 (4 Python worker threads + the driving "
                         "thread over all cores of the process, GIL-serialised; int32 vector add of 64 Ki "
                         "elements via numpy on the worker thread; spin_yield_threshold 10000 = the reference "
                         f"default); p50 {lat_summary(clat)['p50_us']} us",
               "threshold_200": {"tasks_per_s": round(cv2, 2), "latency": lat_summary(clat2),
                                 "note": "spin_yield_threshold=200, the reference test suite's setting "
                                         "(T/test_native.py:13)"},
               "thread_spawn_baseline": None if spawn is None else {
                   "tasks_per_s": round(spawn[0], 2), "latency": lat_summary(spawn[1]),
                   "note": "persistkern.native.ThreadSpawnBaseline launch+wait per task (P/native.py:304-331), "
                           "the vector add on the spawned thread"},
               "threshold_10000_latency": lat_summary(clat)}

    # the denominator is the fastest conventional flow measured, per percentile
    cands = {"work_kernel_grid1": base["grid1"]["launch_plus_sync"]}
    cands.update({k: v["launch_plus_sync"] for k, v in base["floor"].items() if "launch_plus_sync" in v})
    best50 = min(cands, key=lambda k: cands[k]["p50_us"])
    best999 = min(cands, key=lambda k: cands[k]["p99.9_us"])
    lk = lat_summary(done_all)
    noise_sum = noise.summary(done_all, np.percentile(done_all, 50))
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tasks/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t_max / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "configs[1]: empty-task dispatch, 1 persistent CTA per SM on all SMs, "
                               "round-robin single-worker masks", "workers": n, "rounds_per_step": R,
                   "total_rounds": int(units), "threads_per_worker": cfg.threads_per_worker,
                   "cell_stride": cfg.cell_stride, "poll_backoff_ns": cfg.poll_backoff_ns,
                   "poll_mode": cfg.poll_mode, "poll_replicas": cfg.poll_replicas,
                   "poll_spacing_ns": cfg.poll_spacing_ns, "ack_delay_ns": cfg.ack_delay_ns,
                   "ack_adaptive": cfg.ack_adaptive, "payload_path": "tma" if cfg.tma_payload else "lsu",
                   "tma_min_workers": cfg.tma_min_workers,
                   "host_cores_local": pinned, "host_core": pinned_core, "l2": "n/a for the empty task (no payload); payload "
                   "GB/s rotate buffers over >= 4x L2",
                   "timing": "host CLOCK_MONOTONIC per round; max over ranks"},
        "launch_sync_baseline": base,
        **{k: v for k, v in extras.items() if k not in HEADLINE_EXTRAS},
        "payload": payload,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e_value, 1), "unit": "tasks/s",
                "h2d_bytes_per_step": 2 * 8 * cfg.poll_replicas * R, "d2h_bytes_per_step": 3 * 8 * R,
                "note": "Python API session.trigger+session.wait per task (the _lkfast CPython path -> liblk.so), "
                        f"{e2e_rounds} tasks; host<->device traffic per task is the mailbox cells "
                        "themselves: WORK + ack down (8 B x replicas each), WORKING/FINISHED/NOP up (8 B each)"},
        "gpu_launches": world,
        "gpu_launch_note": "one persistent kernel per GPU resident across the timed region; tasks are "
                           "dispatched by mailbox words, not launches",
        "per_rank": per_rank,
        "smid_distinct": len(set(smids)),
        **({"profiled": "run under a profiler: launch list only, not a bench value; session legs that "
                        "call CUDA while resident were skipped"} if prof else {}),
        "clocks": clk.summary(),
        # headline last: the driver keeps the tail of the line
        **{k: extras[k] for k in HEADLINE_EXTRAS if k in extras},
        "host_noise_during_timed_region": noise_sum,
        "latency_us": {"trigger_to_done": lk, "round_trip_with_ack": lat_summary(cyc_all),
                       "init_ms": round(init.cycles / 1e6, 2)},
        "launch_sync_denominator": {"p50_flow": best50, "p50_us": cands[best50]["p50_us"],
                                    "p99.9_flow": best999, "p99.9_us": cands[best999]["p99.9_us"]},
        "speedup_vs_launch_sync_p50": round(cands[best50]["p50_us"] / lk["p50_us"], 2),
        "speedup_vs_launch_sync_p999": round(cands[best999]["p99.9_us"] / lk["p99.9_us"], 2),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["lk", "reference"], default="lk")
    ap.add_argument("--rounds", type=int, default=20_000, help="round trips per step")
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--backoff-ns", type=int, default=0)
    ap.add_argument("--cell-stride", type=int, default=128)
    ap.add_argument("--poll-mode", choices=["gateway", "direct", "hybrid"], default="direct")
    ap.add_argument("--replicas", type=int, default=1)
    ap.add_argument("--spacing-ns", type=int, default=300)
    ap.add_argument("--lsu-payload", action="store_true", help="payload via 128-bit LSU loads, not the TMA ring")
    ap.add_argument("--payload-poll-mode", choices=["gateway", "direct", "hybrid"], default="hybrid")
    ap.add_argument("--interference-poll-mode", choices=["gateway", "direct", "hybrid"], default="hybrid")
    ap.add_argument("--full-rounds", type=int, default=100_000)
    ap.add_argument("--e2e-rounds", type=int, default=100_000)
    ap.add_argument("--base-rounds", type=int, default=100_000)
    ap.add_argument("--pp-rounds", type=int, default=100_000)
    ap.add_argument("--attrib-rounds", type=int, default=300_000, help="tail-attribution rounds (untimed)")
    ap.add_argument("--payload-mib", type=int, nargs="+", default=[1, 2, 4, 8, 16, 32, 64])
    ap.add_argument("--payload-reps", type=int, default=30)
    ap.add_argument("--no-payload", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-interference", action="store_true")
    ap.add_argument("--config0-rounds", type=int, default=20_000)
    ap.add_argument("--no-table2", action="store_true")
    ap.add_argument("--no-lazy", action="store_true")
    ap.add_argument("--no-green", action="store_true")
    ap.add_argument("--no-zero-copy", action="store_true")
    ap.add_argument("--threads", action="store_true",
                    help="configs[4] in one process: a session per visible GPU (or --gpus of them), one "
                         "NUMA-pinned host thread each")
    ap.add_argument("--zc-reps", type=int, default=4000)
    ap.add_argument("--lazy-rounds", type=int, default=200_000)
    ap.add_argument("--drivers", type=int, default=4, help="host threads for the multi-driver throughput extra")
    ap.add_argument("--driver-rounds", type=int, default=100_000)
    ap.add_argument("--lat-workers", type=int, default=16, help="latency partition size (configs[3])")
    ap.add_argument("--interf-rounds", type=int, default=100_000)
    ap.add_argument("--stream-mib", type=int, default=512, help="hbm_stream src (= dst) MiB")
    ap.add_argument("--cpu-budget-s", type=float, default=30.0)
    ap.add_argument("--ref-rounds", type=int, default=0,
                    help="reference arm round trips per step (0: enough for >= 1,000 timed round trips)")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
    elif args.threads:
        if world > 1:
            raise SystemExit("--threads drives every GPU from one process; do not launch it under torchrun")
        run_threads_arm(args)
    else:
        run_lk_arm(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
