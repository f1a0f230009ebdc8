"""GPU sweep of dispatch-latency knobs (C-side closed loop, empty task)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2310_01212_b200 import host, native
from paper_2310_01212_b200.device import WorkDescriptor


def pct(a, q):
    return float(np.percentile(a, q)) / 1e3


def run(label, rounds=20000, mode="rr", **kw):
    cfg = native.NativeConfig(spin_strategy=native.PURE_SPIN, **kw)
    s, _ = native.NativeSession.start(cfg)
    n = s.num_workers
    s.register(WorkDescriptor(slot=0, kind="empty"))
    masks = [1 << i for i in range(n)] if mode == "rr" else [host.full_mask(n)]
    s.bench_roundtrip(masks, 0, 2000)
    _, done, cyc = s.bench_roundtrip(masks, 0, rounds)
    s.dispose()
    s.close()
    print(f"{label:44s} done p50 {pct(done,50):6.2f} p99 {pct(done,99):6.2f} p99.9 {pct(done,99.9):6.2f} "
          f"| cycle p50 {pct(cyc,50):6.2f} p99.9 {pct(cyc,99.9):6.2f}", flush=True)


native.pin_host_thread(0)
pp = native.pingpong(0, 20000)
print("pingpong p50 %.2f p99.9 %.2f" % (pct(pp[100:], 50), pct(pp[100:], 99.9)))
for k, d in ((1, 0), (2, 300), (4, 150), (4, 200), (4, 300), (8, 100), (8, 150)):
    run(f"148 K={k} d={d}", poll_replicas=k, poll_spacing_ns=d or 200)
for k, d in ((1, 0), (4, 200)):
    run(f"1 worker K={k} d={d}", num_workers=1, poll_replicas=k, poll_spacing_ns=d or 200)
    run(f"148 full K={k} d={d}", mode="full", rounds=5000, poll_replicas=k, poll_spacing_ns=d or 200)
run("148 K=4 stride=64", poll_replicas=4, cell_stride=64)
run("148 K=4 threads=1024", poll_replicas=4, threads_per_worker=1024)
