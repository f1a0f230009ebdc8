"""GPU sweep of dispatch-latency knobs (C-side closed loop, empty task).

Prints trigger->FINISHED and full-cycle percentiles per configuration, and the
device-side handling time (to_gpu value seen -> FINISHED issued, globaltimer)
of each worker's last dispatch.
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402


def pct(a, q):
    return float(np.percentile(a, q)) / 1e3


def run(label, rounds=20000, mode="rr", **kw):
    cfg = native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, **kw)
    s, _ = native.NativeSession.start(cfg)
    n = s.num_workers
    s.register(WorkDescriptor(slot=0, kind="empty"))
    masks = [1 << i for i in range(n)] if mode == "rr" else [host.full_mask(n)]
    s.bench_roundtrip(masks, 0, 2000)
    _, done, cyc = s.bench_roundtrip(masks, 0, rounds)
    t = s.last_timeline().astype(np.int64)
    s.dispose()
    s.close()
    dev = np.median(t[:, 7] - t[:, 5])
    print(f"{label:40s} done p50 {pct(done,50):6.2f} p99 {pct(done,99):6.2f} p99.9 {pct(done,99.9):6.2f} "
          f"| cycle p50 {pct(cyc,50):6.2f} p99.9 {pct(cyc,99.9):6.2f} | dev {dev:5.0f} cyc", flush=True)


native.pin_host_thread(0)
pp = native.pingpong(0, 20000)
print("pingpong p50 %.2f p99.9 %.2f" % (pct(pp[100:], 50), pct(pp[100:], 99.9)))
run("148 rr direct")
