"""Where the Python API's per-task time goes: C loop (lk_bench_roundtrip) vs
a bare ctypes loop (raw handles, no wrapper) vs session.trigger+session.wait."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import _lib, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None))
n = s.num_workers
w = WorkDescriptor(slot=0, kind="empty")
s.register(w, 1)
N = 100_000
for trial in range(3):
    # C loop
    masks = np.zeros((n, s.nwords), dtype=np.uint64)
    for i in range(n):
        masks[i, i // 64] = np.uint64(1 << (i % 64))
    cyc = np.zeros(N, dtype=np.uint64)
    t0 = time.perf_counter_ns()
    _lib.check(s._lib.lk_bench_roundtrip(s._h, masks.tobytes(), n, s.nwords, 0, N, None, None, cyc.ctypes.data))
    c_ns = (time.perf_counter_ns() - t0) / N
    # bare ctypes
    mb = [(1 << i).to_bytes(8 * s.nwords, "little") for i in range(n)]
    u = C.c_uint64()
    ur = C.byref(u)
    trig, wait, h, nw = s._raw_trigger, s._raw_wait, s._h, s.nwords
    t0 = time.perf_counter_ns()
    for k in range(N):
        m = mb[k % n]
        trig(h, m, nw, 0, None, ur)
        wait(h, m, nw, ur)
    raw_ns = (time.perf_counter_ns() - t0) / N
    # the CPython fast object directly (no Python method frame around it)
    f = s._fast
    t0 = time.perf_counter_ns()
    for k in range(N):
        m = 1 << (k % n)
        f.trigger(m, w)
        f.wait(m)
    fast_ns = (time.perf_counter_ns() - t0) / N
    s.timings.clear()
    # API
    t0 = time.perf_counter_ns()
    for k in range(N):
        m = 1 << (k % n)
        s.trigger(m, w)
        s.wait(m)
    api_ns = (time.perf_counter_ns() - t0) / N
    s.timings.clear()
    print(f"per task: C loop {c_ns:7.0f} ns | bare ctypes {raw_ns:7.0f} ns | _lkfast direct {fast_ns:7.0f} ns | "
          f"API {api_ns:7.0f} ns", flush=True)
s.dispose()
s.close()
