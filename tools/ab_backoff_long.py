"""DIRECT-mode idle-poll backoff (poll_backoff_ns) at long values: round 1
measured 0-400 ns (every step slower); a HYBRID poller experiment suggested
0.7-1.5 us sleeps shorten the link's round trip by taking reads out of
flight.  148-worker round robin and one worker, from C, interleaved."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})


def q(x):
    return f"{np.percentile(x, 50)/1e3:5.3f}/{np.percentile(x, 99.9)/1e3:5.2f}"


for rep in range(3):
    for b in [int(x) for x in sys.argv[1:]] or [0, 700, 1000, 1500, 2500]:
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN,
                                                              poll_backoff_ns=b))
        s.register(WorkDescriptor(slot=0, kind="empty"))
        rr = [1 << i for i in range(s.num_workers)]
        s.bench_roundtrip(rr, 0, 20000)
        _, d, c = s.bench_roundtrip(rr, 0, 200000)
        _, d1, c1 = s.bench_roundtrip([1], 0, 50000)
        print(f"rep {rep} backoff {b:5d}: rr148 {q(d)} cyc {q(c)} {200000 / (c.sum() / 1e9) / 1e3:.0f}k/s | "
              f"one {q(d1)} cyc {q(c1)}", flush=True)
        s.dispose()
        s.close()
