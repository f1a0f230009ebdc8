"""GATEWAY mode: event-ring replicas (poll_replicas 1/2/4, the gateway warp's
staggered ring loads) for full-mask and round-robin empty-task loops."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
res = {}
for trial in range(3):
    for k in (1, 2, 4):
        for sp in ((300,) if k == 1 else (150, 300)):
            s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, poll_mode="gateway",
                                                                  poll_replicas=k, poll_spacing_ns=sp))
            n = s.num_workers
            s.register(WorkDescriptor(slot=0, kind="empty"))
            for pat, masks in (("full", [host.full_mask(n)]), ("rr148", [1 << i for i in range(n)])):
                s.bench_roundtrip(masks, 0, 2000)
                _, done, cyc = s.bench_roundtrip(masks, 0, 20000)
                res.setdefault((pat, k, sp), []).append((np.median(done) / 1e3, np.median(cyc) / 1e3))
            s.dispose()
            s.close()
for key in sorted(res):
    a = np.median(np.array(res[key]), axis=0)
    print(f"{key[0]:6s} replicas {key[1]} spacing {key[2]:3d}: done p50 {a[0]:.3f} | cycle p50 {a[1]:.3f} us", flush=True)
