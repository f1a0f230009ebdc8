"""The reference's default task -- WorkDescriptor(slot), a busy_loop of 0
iterations -- against kind="empty": 148-worker round robin, C loop."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN))
n = s.num_workers
masks = [1 << i for i in range(n)]
for trial in range(3):
    for name, w in (("empty", WorkDescriptor(slot=0, kind="empty")), ("busy(0)", WorkDescriptor(slot=1)),
                    ("busy(1)", WorkDescriptor(slot=2, iterations=1))):
        s.register(w)
        s.bench_roundtrip(masks, w.slot, 5000)
        _, done, cyc = s.bench_roundtrip(masks, w.slot, 60000)
        print(f"{name:8s} done p50 {np.median(done) / 1e3:.3f} | cycle p50 {np.median(cyc) / 1e3:.3f} us", flush=True)
s.dispose()
s.close()
