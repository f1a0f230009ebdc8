"""Where does the p99.9 tail of the empty round trip come from?  Times of the
slow rounds (cumulative cycle time) and their spacing: a fixed period points
at a host timer tick, not at the GPU."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

import os  # noqa: E402
native.pin_host_thread(0)
cores = sorted(os.sched_getaffinity(0))
os.sched_setaffinity(0, {cores[-1]})
if "fifo" in sys.argv:
    os.sched_setscheduler(0, os.SCHED_FIFO, os.sched_param(50))
    print("SCHED_FIFO 50")
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN))
n = s.num_workers
s.register(WorkDescriptor(slot=0, kind="empty"))
masks = [1 << i for i in range(n)]
s.bench_roundtrip(masks, 0, 5000)
_, done, cyc = s.bench_roundtrip(masks, 0, 400000)
s.dispose()
s.close()
t = np.cumsum(cyc.astype(np.int64)) / 1e6   # ms since start (ack-inclusive cycles back to back)
thr = 4000
slow = np.nonzero(done > thr)[0]
print(f"rounds {len(done)}, p50 {np.median(done)/1e3:.2f} us, p99.9 {np.percentile(done, 99.9)/1e3:.2f} us, "
      f"slow(>{thr/1e3:.0f}us) {len(slow)} over {t[-1]:.0f} ms -> {len(slow)/t[-1]*1e3:.0f} per s")
if len(slow) > 3:
    gaps = np.diff(t[slow])
    print("gap between slow rounds (ms): p10 %.2f p50 %.2f p90 %.2f" % tuple(np.percentile(gaps, [10, 50, 90])))
    hist, edges = np.histogram(gaps, bins=[0, 0.5, 1, 2, 3, 3.9, 4.1, 5, 8, 1e9])
    print("gap histogram:", {f"{edges[i]:.1f}-{edges[i+1]:.1f}": int(h) for i, h in enumerate(hist)})
    print("slow round latency (us): p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(done[slow] / 1e3, [50, 90, 100])))
# which workers are slow? (device-side cause would cluster on SMs)
w = slow % n
print("distinct workers among slow rounds:", len(set(w.tolist())), "of", n)
