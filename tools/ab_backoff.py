"""Idle-poll backoff (poll_backoff_ns: __nanosleep between a worker's cell
loads) against link contention: 148 workers round robin, C loop,
interleaved trials, default ack delay."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
vals = [int(x) for x in sys.argv[1:]] or [0, 50, 100, 200, 400]
res = {}
for trial in range(3):
    for b in vals:
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, poll_backoff_ns=b))
        n = s.num_workers
        s.register(WorkDescriptor(slot=0, kind="empty"))
        masks = [1 << i for i in range(n)]
        s.bench_roundtrip(masks, 0, 5000)
        _, done, cyc = s.bench_roundtrip(masks, 0, 100000)
        s.dispose()
        s.close()
        res.setdefault(b, []).append((np.percentile(done, 50), np.percentile(done, 99.9), np.percentile(cyc, 50)))
for b in vals:
    a = np.median(np.array(res[b]), axis=0) / 1e3
    print(f"backoff {b:4d} ns: done p50 {a[0]:.3f} p99.9 {a[1]:.3f} | cycle p50 {a[2]:.3f} us", flush=True)
