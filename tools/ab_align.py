"""LK_CF_ALIGN A/B: idle polls timed to the latest publish + the host's
reaction time, against free-running polls.  The option was removed after
this A/B measured it worse from C; the tool records the
run and needs that experimental build (git history) to execute.  C loops (148 round robin, 4
round robin, one worker) and the Python API round robin; interleaved."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
res = {}
for trial in range(3):
    for name, kw in (("free", {}), ("align", dict(align_polls=True))):
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, **kw))
        n = s.num_workers
        w = WorkDescriptor(slot=0, kind="empty")
        s.register(w)
        for pat, masks in (("rr148", [1 << i for i in range(n)]), ("rr4", [1, 2, 4, 8]), ("single", [1])):
            s.bench_roundtrip(masks, 0, 5000)
            _, done, cyc = s.bench_roundtrip(masks, 0, 60000)
            res.setdefault((pat, name), []).append((np.percentile(done, 50) / 1e3, np.percentile(done, 99.9) / 1e3,
                                                    np.percentile(cyc, 50) / 1e3, 60000 / (cyc.sum() / 1e9) / 1e3))
        N = 40000
        for k in range(3000):
            m = 1 << (k % n)
            s.trigger(m, w)
            s.wait(m)
        t0 = time.perf_counter_ns()
        for k in range(N):
            m = 1 << (k % n)
            s.trigger(m, w)
            s.wait(m)
        dt = time.perf_counter_ns() - t0
        s.timings.clear()
        res.setdefault(("py-rr148", name), []).append((np.nan, np.nan, dt / N / 1e3, N / (dt / 1e9) / 1e3))
        s.dispose()
        s.close()
for key in sorted(res):
    a = np.nanmedian(np.array(res[key], dtype=float), axis=0)
    print(f"{key[0]:9s} {key[1]:6s} done p50 {a[0]:.3f} p99.9 {a[1]:.3f} | cycle p50 {a[2]:.3f} us | {a[3]:.0f}k tasks/s",
          flush=True)
