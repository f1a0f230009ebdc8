"""Two builds of liblk.so compared in alternating processes: pass the
library directory as argv[1]; prints the 148-worker round-robin C-loop
cycle.  (Used for host-side reorderings that need a rebuild to A/B.)"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN))
n = s.num_workers
s.register(WorkDescriptor(slot=0, kind="empty"))
m = [1 << i for i in range(n)]
s.bench_roundtrip(m, 0, 20000)
_, done, cyc = s.bench_roundtrip(m, 0, 200000)
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'build'}: done p50 {np.median(done) / 1e3:.3f} cycle p50 "
      f"{np.median(cyc) / 1e3:.3f} us", flush=True)
s.dispose()
s.close()
