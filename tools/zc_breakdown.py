"""Where a zero-copy (host-mapped) dispatch's time goes, against the same
4-byte vector add on device buffers: device globaltimer stamps of worker 0's
dispatch (value seen, work begin, work end, FINISHED issued) and host
trigger->done, for several variants."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, HostBuffer, WorkDescriptor  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
EXP = 0x80000000


def run(label, cfg_flags_extra, host_bufs, n=1, reps=3000):
    cfg = native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, timeline=True)
    s, _ = native.NativeSession.start(cfg)
    if cfg_flags_extra:
        s._lib  # noqa
    if host_bufs:
        a, b, o = HostBuffer(4 * n), HostBuffer(4 * n), HostBuffer(4 * n)
    else:
        a, b, o = DeviceBuffer(4 * n), DeviceBuffer(4 * n), DeviceBuffer(4 * n)
    w = WorkDescriptor(slot=5, kind="vector_add_i32", data_in_ref=(a, b), data_out_ref=o)
    s.register(w, 1)
    rows = []
    done_all = []
    for r in range(reps):
        _, done, _ = s.bench_roundtrip([1], 5, 1)
        tl = s.last_timeline()[0].astype(np.int64)
        if r >= 200:
            rows.append((tl[1] - tl[0], tl[2] - tl[1], tl[3] - tl[2]))
            done_all.append(done[0])
    m = np.median(np.array(rows), axis=0)
    print(f"{label:28s} n={n:6d}: host trigger->done p50 {np.median(done_all)/1e3:6.2f} us | seen->begin "
          f"{m[0]/1e3:5.2f} | begin->end {m[1]/1e3:5.2f} | end->FINISHED {m[2]/1e3:5.2f} us", flush=True)
    s.dispose()
    s.close()


import ctypes  # noqa: E402,F401
orig = native.NativeConfig.to_c


def with_flags(extra):
    def to_c(self):
        c = orig(self)
        c.flags |= extra
        return c
    return to_c


for n in (1, 1024, 16384):
    native.NativeConfig.to_c = orig
    run("device buffers", 0, False, n)
    run("host buffers", 0, True, n)
    native.NativeConfig.to_c = with_flags(EXP)
    run("host buffers, no acq fence", EXP, True, n)
native.NativeConfig.to_c = orig
