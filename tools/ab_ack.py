"""Ack-phase polling variants, interleaved: after publishing FINISHED a worker
(a) reloads its cell at once (ack_delay_ns=0), (b) waits a fixed ack_delay_ns before its
first reload, (c) starts from ack_delay_ns and adapts it (the default).  148 workers, round robin, C loop."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
variants = {"no-delay": dict(ack_delay_ns=0)}
for d in (150, 200, 250, 300, 400):
    variants[f"fixed{d}"] = dict(ack_delay_ns=d, ack_adaptive=False)
for d in (150, 300, 600):
    variants[f"adapt{d}"] = dict(ack_delay_ns=d)
res = {k: [] for k in variants}
for trial in range(3):
    for name, kw in variants.items():
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, **kw))
        n = s.num_workers
        s.register(WorkDescriptor(slot=0, kind="empty"))
        masks = [1 << i for i in range(n)]
        s.bench_roundtrip(masks, 0, 5000)
        _, done, cyc = s.bench_roundtrip(masks, 0, 100000)
        s.dispose()
        s.close()
        res[name].append((np.percentile(done, 50) / 1e3, np.percentile(cyc, 50) / 1e3, np.mean(cyc) / 1e3,
                          np.percentile(done, 99.9) / 1e3))
for name, r in res.items():
    a = np.median(np.array(r), axis=0)
    print(f"{name:10s} done p50 {a[0]:.3f} | cycle p50 {a[1]:.3f} mean {a[2]:.3f} -> {1e6 / a[2] / 1e3:.0f}k tasks/s "
          f"| done p99.9 {a[3]:.3f} us", flush=True)
