"""Host time inside the C loop: trigger call start -> WORK word written
(checks + post), per worker's last dispatch (lk_last_host_times), after a
148-worker round-robin lk_bench_roundtrip run."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN))
n = s.num_workers
s.register(WorkDescriptor(slot=0, kind="empty"))
masks = [1 << i for i in range(n)]
for rep in range(3):
    trig, done, cyc = s.bench_roundtrip(masks, 0, 50000)
    h = s.last_host_times().astype(np.int64)
    pre = h[:, 1] - h[:, 0]
    print(f"trigger start -> WORK written: p50 {np.median(pre):.0f} ns p90 {np.percentile(pre, 90):.0f} ns | "
          f"post alone p50 {np.median(trig):.0f} ns | WORK written -> FINISHED seen p50 "
          f"{np.median(h[:, 2] - h[:, 1]) / 1e3:.3f} us | cycle p50 {np.median(cyc) / 1e3:.3f} us", flush=True)
s.dispose()
s.close()
