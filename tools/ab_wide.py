"""Full-mask (148-worker) empty dispatch by poll mode and poll ordering
(acquire vs relaxed), sessions interleaved: trigger call, trigger->done and
the full cycle, p50/p99.9 us."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})


def q(x):
    return f"{np.percentile(x, 50)/1e3:5.2f}/{np.percentile(x, 99.9)/1e3:5.2f}"


modes = sys.argv[1:] or ["direct", "gateway", "hybrid"]
for rep in range(2):
    for mode in modes:
        for acq in (True, False):
            s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN,
                                                                  poll_mode=mode, acquire_poll=acq))
            s.register(WorkDescriptor(slot=0, kind="empty"))
            full = host.full_mask(s.num_workers)
            s.bench_roundtrip([full], 0, 2000)
            t, d, c = s.bench_roundtrip([full], 0, 30000)
            print(f"rep {rep} {mode:8s} acquire={int(acq)} trigger call {q(t)} done {q(d)} cycle {q(c)}", flush=True)
            s.dispose()
            s.close()
