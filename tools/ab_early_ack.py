"""Historical A/B (env LK_EARLY_ACK, since removed: early acks are the default)
of DIRECT-mode wide waits that ack each
worker the moment its FINISHED is seen, instead of all after the last.
Full-mask and 16-worker dispatch, 64 MiB saxpy e2e on direct vs gateway."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})


def q(x):
    return f"{np.percentile(x, 50)/1e3:5.2f}/{np.percentile(x, 99.9)/1e3:5.2f}"


out = []
for mode in ("direct", "gateway"):
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN,
                                                          poll_mode=mode))
    s.register(WorkDescriptor(slot=0, kind="empty"))
    full = host.full_mask(s.num_workers)
    s.bench_roundtrip([full], 0, 2000)
    _, d, c = s.bench_roundtrip([full], 0, 20000)
    out.append(f"{mode} full {q(d)} cyc {q(c)}")
    _, d, c = s.bench_roundtrip([0xFFFF], 0, 20000)
    out.append(f"16w {q(d)} cyc {q(c)}")
    r = bench.measure_payload(s, "saxpy_f32", [64], 16, 4 * bench.L2_BYTES)["64MiB"]
    out.append(f"saxpy64 {r['gbs_device']:.0f}/{r['gbs_e2e']:.0f}")
    s.dispose()
    s.close()
print(f"early_ack={os.environ.get('LK_EARLY_ACK', '0')}: " + " | ".join(out), flush=True)
