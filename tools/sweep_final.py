"""Round-1 latency sweep for profiles/: poll modes x worker counts x mask
shapes, plus the ping-pong floor and launch+sync, on one box."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402


def pct(a, q):
    return float(np.percentile(a, q)) / 1e3


def line(label, done, cyc=None):
    s = f"{label:42s} p50 {pct(done,50):6.2f} p90 {pct(done,90):6.2f} p99 {pct(done,99):6.2f} p99.9 {pct(done,99.9):6.2f}"
    if cyc is not None:
        s += f" | cycle p50 {pct(cyc,50):6.2f} -> {len(cyc)/(cyc.sum()/1e9)/1e3:7.1f}k tasks/s"
    print(s, flush=True)


native.pin_host_thread(0)
import os  # noqa: E402
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
pp = native.pingpong(0, 50000)[100:]
line("ping-pong floor (1 poller)", pp)
for mode in ("direct", "hybrid", "gateway"):
    for nw in (16, 148):
        s, _ = native.NativeSession.start(native.NativeConfig(spin_strategy=native.PURE_SPIN, poll_mode=mode,
                                                              num_workers=nw))
        s.register(WorkDescriptor(slot=0, kind="empty"))
        rr = [1 << i for i in range(nw)]
        s.bench_roundtrip(rr, 0, 5000)
        _, done, cyc = s.bench_roundtrip(rr, 0, 100000)
        line(f"{mode:8s} {nw:3d} workers round robin", done, cyc)
        _, done, cyc = s.bench_roundtrip([host.full_mask(nw)], 0, 20000)
        line(f"{mode:8s} {nw:3d} workers full mask", done, cyc)
        if nw == 148:
            s.bench_roundtrip([1], 0, 5000)
            _, done, cyc = s.bench_roundtrip([1], 0, 100000)
            line(f"{mode:8s} {nw:3d} workers, one re-triggered", done, cyc)
        s.dispose()
        s.close()
b = native.LaunchSyncBaseline()
w = WorkDescriptor(slot=0, kind="empty")
b.bench(w, 1000, 1)
_, tot = b.bench(w, 100000, 1)
line("cudaLaunchKernel + cudaStreamSynchronize, grid 1", tot)
_, tot = b.bench(w, 100000, 148)
line("cudaLaunchKernel + cudaStreamSynchronize, grid 148", tot)
b.close()
