"""Where a full-mask (148-worker) empty dispatch's time goes: device
globaltimer stamps (LK_CF_TIMELINE) of the gateway forward, each worker's
value seen and FINISHED issued, against the host's trigger->done.  The
device part is first forward -> last FINISHED issued; the rest is the two
link crossings and the host's scan."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
for mode in ("gateway", "direct"):
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN,
                                                          poll_mode=mode, timeline=True))
    s.register(WorkDescriptor(slot=0, kind="empty"))
    full = host.full_mask(s.num_workers)
    s.bench_roundtrip([full], 0, 500)
    rows = []
    for r in range(3000):
        t, d, c = s.bench_roundtrip([full], 0, 1)
        tl = s.last_timeline().astype(np.int64)
        seen, fin = tl[:, 0], tl[:, 3]
        t0 = tl[:, 4].min() if mode == "gateway" else seen.min()
        rows.append((d[0], c[0], t[0], seen.max() - t0, np.median(seen) - t0, fin.max() - t0,
                     np.median(fin - seen), fin.max() - fin.min()))
    a = np.median(np.array(rows, dtype=np.float64), axis=0) / 1e3
    print(f"{mode:8s} host trigger->done {a[0]:5.2f} cycle {a[1]:5.2f} (trigger call {a[2]:4.2f}) | device: "
          f"{'forward' if mode == 'gateway' else 'first seen'} -> last seen {a[3]:4.2f} (median {a[4]:4.2f}) -> "
          f"last FINISHED issued {a[5]:4.2f} | per-worker seen->FINISHED {a[6]:4.2f} | FINISHED spread {a[7]:4.2f} us",
          flush=True)
    s.dispose()
    s.close()
