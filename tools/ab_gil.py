"""_lkfast: keep the GIL across lk_trigger (direct, no lazy ack) or release
it, on the Python-API round-robin loop of bench.py's e2e; one session,
interleaved trials."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200 import _lib, _lkfast  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402
from paper_2310_01212_b200.host import PHASE_TRIGGER, PHASE_WAIT, PhaseTiming  # noqa: E402

native.pin_host_thread(0)
import os  # noqa: E402
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN))
n = s.num_workers
w = WorkDescriptor(slot=0, kind="empty")
raw = _lib.raw()
addr = lambda fn: C.cast(fn, C.c_void_p).value  # noqa: E731


def fast(keep):
    return _lkfast.Fast(s._h.value, s.nwords, addr(raw.lk_trigger), addr(raw.lk_wait), s._staged, s._mask_cache,
                        s._timings._rows, 1 << n, PhaseTiming, WorkDescriptor, PHASE_TRIGGER, PHASE_WAIT, keep)


for k in range(3000):
    m = 1 << (k % n)
    s.trigger(m, w)
    s.wait(m)
N = 100_000
res = {True: [], False: []}
for trial in range(4):
    for keep in (True, False):
        s._fast = fast(keep)
        t0 = time.perf_counter_ns()
        for k in range(N):
            m = 1 << (k % n)
            s.trigger(m, w)
            s.wait(m)
        res[keep].append(N / ((time.perf_counter_ns() - t0) / 1e9) / 1e3)
        s.timings.clear()
for keep, v in res.items():
    print(f"keep_gil={keep}: {np.median(v):.1f}k tasks/s  {[round(x, 1) for x in v]}", flush=True)
s.dispose()
s.close()
