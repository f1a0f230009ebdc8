"""cell_stride (bytes between workers' to_gpu cells) A/B: 148-worker round
robin and full-mask dispatch on DIRECT sessions, interleaved."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})


def q(x):
    return f"{np.percentile(x, 50)/1e3:5.3f}/{np.percentile(x, 99.9)/1e3:5.2f}"


strides = [int(a) for a in sys.argv[1:]] or [128, 64, 32]
for rep in range(2):
    for cs in strides:
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN,
                                                              cell_stride=cs))
        s.register(WorkDescriptor(slot=0, kind="empty"))
        n = s.num_workers
        rr = [1 << i for i in range(n)]
        s.bench_roundtrip(rr, 0, 20000)
        _, d, c = s.bench_roundtrip(rr, 0, 200000)
        full = host.full_mask(n)
        s.bench_roundtrip([full], 0, 2000)
        t, fd, fc = s.bench_roundtrip([full], 0, 20000)
        print(f"rep {rep} cell_stride {cs:3d}: rr {q(d)} cyc {q(c)} | full trigger call {q(t)} done {q(fd)} "
              f"cyc {q(fc)}", flush=True)
        s.dispose()
        s.close()
