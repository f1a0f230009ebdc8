"""Payload dispatch latency: full-mask saxpy through the C loop and the Python
API, with each worker's device-side cycles (value seen -> FINISHED issued)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "direct"
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, poll_mode=mode))
print("poll mode", mode)
n = s.num_workers
full = host.full_mask(n)
s.register(WorkDescriptor(slot=0, kind="empty"))
_, done, _ = s.bench_roundtrip([full], 0, 3000)
print(f"empty full-mask C loop: done p50 {np.median(done)/1e3:.2f} us")
for kib in (64, 1024, 16384, 65536):
    el = kib * 256
    x, y = DeviceBuffer(4 * el), DeviceBuffer(4 * el)
    w = WorkDescriptor(slot=5, kind="saxpy_f32", data_in_ref=(x, y), data_out_ref=y, alpha=1.0)
    s.register(w, full)
    trig, done, cyc = s.bench_roundtrip([full], 5, 500)
    t = s.last_timeline().astype(np.int64)
    py = []
    for _ in range(300):
        a = time.perf_counter_ns()
        s.trigger(full, w)
        s.wait(full)
        py.append(time.perf_counter_ns() - a)
    print(f"saxpy {kib:6d} KiB: C trig p50 {np.median(trig)/1e3:6.2f} done p50 {np.median(done)/1e3:7.2f} "
          f"cycle p50 {np.median(cyc)/1e3:7.2f} | python e2e p50 {np.median(py)/1e3:7.2f} us | "
          f"dev cycles seen->begin {np.median(t[:,6]-t[:,5]):.0f} begin->fin {np.median(t[:,7]-t[:,6]):.0f} "
          f"| span {(t[:,2].max()-t[:,1].min())/1e3:.2f} us", flush=True)
    x.free(); y.free()
s.dispose()
s.close()
