"""status_stride (bytes between from_gpu status cells) vs the host's scan of
148 cells: full-mask and round-robin C loops, direct and gateway modes."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
res = {}
for trial in range(3):
    for mode in ("direct", "gateway"):
        for stride in (128, 64, 16):
            s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, poll_mode=mode,
                                                                  status_stride=stride))
            n = s.num_workers
            s.register(WorkDescriptor(slot=0, kind="empty"))
            for pat, masks in (("full", [host.full_mask(n)]), ("rr148", [1 << i for i in range(n)])):
                s.bench_roundtrip(masks, 0, 2000)
                _, done, cyc = s.bench_roundtrip(masks, 0, 20000)
                res.setdefault((mode, pat, stride), []).append((np.median(done) / 1e3, np.median(cyc) / 1e3))
            s.dispose()
            s.close()
for key in sorted(res):
    a = np.median(np.array(res[key]), axis=0)
    print(f"{key[0]:8s} {key[1]:6s} status_stride {key[2]:3d}: done p50 {a[0]:.3f} us | cycle p50 {a[1]:.3f} us",
          flush=True)
