"""Interleaved A/B of poll modes on the bench's configs[1] loop (148 workers,
empty task, round robin)."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
modes = sys.argv[1:] or ["direct", "hybrid"]
res = {m: [] for m in modes}
for trial in range(4):
    for m in modes:
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, poll_mode=m))
        s.register(WorkDescriptor(slot=0, kind="empty"))
        rr = [1 << i for i in range(s.num_workers)]
        s.bench_roundtrip(rr, 0, 5000)
        _, done, cyc = s.bench_roundtrip(rr, 0, 200000)
        res[m].append((np.median(done) / 1e3, np.percentile(done, 99.9) / 1e3, len(cyc) / (cyc.sum() / 1e9) / 1e3))
        s.dispose()
        s.close()
for m, v in res.items():
    a = np.array(v)
    print(f"{m:8s} p50 {np.median(a[:,0]):.3f} us  p99.9 {np.median(a[:,1]):.3f} us  {np.median(a[:,2]):.1f}k tasks/s   "
          f"trials {[tuple(round(x, 2) for x in t) for t in v]}", flush=True)
