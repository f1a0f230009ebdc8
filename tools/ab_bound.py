"""session.trigger/wait bound to the CPython fast path's methods (no Python
frame) vs the class methods wrapping the same fast object: the Python-API
round-robin loop of bench.py's e2e, one session, interleaved trials."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN))
n = s.num_workers
w = WorkDescriptor(slot=0, kind="empty")
rr = [1 << i for i in range(n)]
for k in range(3000):
    s.trigger(rr[k % n], w)
    s.wait(rr[k % n])
N = 100_000
res = {"bound": [], "wrapped": []}
for trial in range(4):
    for mode in ("bound", "wrapped"):
        s._bind_fast()
        if mode == "wrapped":   # keep the fast object, drop the instance bindings
            s.__dict__.pop("trigger")
            s.__dict__.pop("wait")
        t0 = time.perf_counter_ns()
        for k in range(N):
            m = rr[k % n]
            s.trigger(m, w)
            s.wait(m)
        res[mode].append(N / ((time.perf_counter_ns() - t0) / 1e9) / 1e3)
        s.timings.clear()
for mode, v in res.items():
    print(f"{mode:8s}: {np.median(v):.1f}k tasks/s  {[round(x, 1) for x in v]}", flush=True)
s.dispose()
s.close()
