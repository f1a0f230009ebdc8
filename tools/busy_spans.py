"""Table II's LK/Wait vs BASE/Wait gap for busy_loop(20000): the loop's own
device time in the persistent kernel (clock64 stamps around it, cached fast
path and general path) against the baseline kernel's device time (CUDA
events, back-to-back launches) and its launch+sync, grid 1 and 148."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
IT = 20000
GHZ = 1.965
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN))
n = s.num_workers
w = WorkDescriptor(slot=3, iterations=IT)
for mask, name in ((1, "one worker"), (host.full_mask(n), "all workers")):
    s.register(w, mask)
    d_us, h_us = [], []
    for r in range(60):
        _, done, _ = s.bench_roundtrip([mask], 3, 1)
        tl = s.last_timeline().astype(np.int64)
        if r >= 10:
            d_us.append(np.median(tl[:, 7][tl[:, 7] > 0] - tl[:, 6][tl[:, 7] > 0]) / GHZ / 1e3 if mask != 1
                        else (tl[0, 7] - tl[0, 6]) / GHZ / 1e3)
            h_us.append(done[0] / 1e3)
    print(f"LK {name}: device begin->FINISHED {np.median(d_us):7.2f} us | host trigger->done {np.median(h_us):7.2f} us",
          flush=True)
s.dispose()
s.close()
b = native.LaunchSyncBaseline()
for grid in (1, 148):
    ms = b.time_kernel(w, 50, grid)
    _, tot = b.bench(w, 50, grid)
    print(f"baseline grid {grid}: device {ms * 1e3:7.2f} us per launch (events) | launch+sync {np.median(tot) / 1e3:7.2f} us",
          flush=True)
b.close()
