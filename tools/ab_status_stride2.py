"""status_stride 64 vs 32 on every loop the bench reports: 148-worker round
robin and one worker (direct), full mask (direct, gateway), 64 MiB saxpy
e2e (gateway); sessions interleaved, 3 trials."""
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
    return f"{np.percentile(x, 50)/1e3:5.3f}/{np.percentile(x, 99.9)/1e3:5.2f}"


for rep in range(3):
    for stride in (64, 32):
        out = []
        for mode in ("direct", "gateway"):
            s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN,
                                                                  poll_mode=mode, status_stride=stride))
            s.register(WorkDescriptor(slot=0, kind="empty"))
            n = s.num_workers
            full = host.full_mask(n)
            if mode == "direct":
                rr = [1 << i for i in range(n)]
                s.bench_roundtrip(rr, 0, 20000)
                _, d, c = s.bench_roundtrip(rr, 0, 200000)
                out.append(f"rr {q(d)} cyc {q(c)} {200000 / (c.sum() / 1e9) / 1e3:.0f}k/s")
                _, d, c = s.bench_roundtrip([1], 0, 50000)
                out.append(f"one {q(d)}")
            s.bench_roundtrip([full], 0, 2000)
            _, d, c = s.bench_roundtrip([full], 0, 20000)
            out.append(f"{mode} full {q(d)} cyc {q(c)}")
            if mode == "gateway":
                r = bench.measure_payload(s, "saxpy_f32", [64], 16, 4 * bench.L2_BYTES)["64MiB"]
                out.append(f"saxpy64 {r['gbs_device']:.0f}/{r['gbs_e2e']:.0f}")
            s.dispose()
            s.close()
        print(f"rep {rep} stride {stride}: " + " | ".join(out), flush=True)
