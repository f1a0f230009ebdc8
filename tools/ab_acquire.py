"""A/B: ld.acquire.sys polls (LK_CF_ACQUIRE_POLL) against ld.relaxed.sys, on
the configs[1] loop (148 workers round robin, empty task, from C), on one
worker re-triggered back to back, and on a 4-byte zero-copy vector add (where
the acquire poll replaces the sys-scope fence).  Sessions interleaved."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import HostBuffer, WorkDescriptor  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
R = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000


def q(x):
    return f"p50 {np.percentile(x, 50)/1e3:5.3f} p99 {np.percentile(x, 99)/1e3:5.3f} p99.9 {np.percentile(x, 99.9)/1e3:5.3f}"


for rep in range(3):
    for acq in (False, True):
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN,
                                                              acquire_poll=acq))
        s.register(WorkDescriptor(slot=0, kind="empty"))
        rr = [1 << i for i in range(s.num_workers)]
        s.bench_roundtrip(rr, 0, 20_000)
        _, d, c = s.bench_roundtrip(rr, 0, R)
        _, d1, c1 = s.bench_roundtrip([1], 0, R // 4)
        ha, hb, ho = HostBuffer(4), HostBuffer(4), HostBuffer(4)
        s.register(WorkDescriptor(slot=1, kind="vector_add_i32", data_in_ref=(ha, hb), data_out_ref=ho), 1)
        s.bench_roundtrip([1], 1, 500)
        _, dz, cz = s.bench_roundtrip([1], 1, 5000)
        print(f"rep {rep} acquire={int(acq)} rr done {q(d)} cyc {q(c)} | one done {q(d1)} | zc4B done {q(dz)}",
              flush=True)
        s.dispose()
        s.close()
