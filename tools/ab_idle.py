"""Idle delay (the first poll after the NOP that closes a handshake; adaptive,
from the given start) vs how soon the host re-triggers the same worker: a single-worker C loop, a
single-worker Python-API loop, 4-worker and 148-worker round robin.
ack_delay_ns stays at its default; interleaved trials."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
idles = [int(x) for x in sys.argv[1:]] or [0, 300, 600]
res = {}
for trial in range(3):
    for idle in idles:
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, idle_delay_ns=idle))
        n = s.num_workers
        w = WorkDescriptor(slot=0, kind="empty")
        s.register(w)
        for pat, masks in (("single", [1]), ("rr4", [1, 2, 4, 8]), ("rr148", [1 << i for i in range(n)])):
            s.bench_roundtrip(masks, 0, 3000)
            _, done, cyc = s.bench_roundtrip(masks, 0, 50000)
            res.setdefault((pat, idle), []).append((np.percentile(done, 50) / 1e3, np.percentile(cyc, 50) / 1e3))
        N = 50000
        for k in range(2000):
            s.trigger(1, w)
            s.wait(1)
        t0 = time.perf_counter_ns()
        for k in range(N):
            s.trigger(1, w)
            s.wait(1)
        per = (time.perf_counter_ns() - t0) / N / 1e3
        s.timings.clear()
        res.setdefault(("py-single", idle), []).append((float("nan"), per))
        s.dispose()
        s.close()
for (pat, idle), r in sorted(res.items()):
    a = np.nanmedian(np.array(r), axis=0)
    print(f"{pat:9s} idle {idle:4d} ns: done p50 {a[0]:.3f} | cycle {a[1]:.3f} us -> {1e3 / a[1]:.0f}k tasks/s",
          flush=True)
