"""block_reduce_f32 device GB/s by size and ring depth (bench.measure_payload,
GATEWAY session, L2-cold by rotation), interleaved trials.

    python tools/reduce_sizes.py [stages ...]
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402

native.pin_host_thread(0)
stages = [int(x) for x in sys.argv[1:]] or [6]
sizes = [16, 64, 256, 1024]
res = {}
for trial in range(2):
    for st in stages:
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway", ring_stages=st))
        r = bench.measure_payload(s, "block_reduce_f32", sizes, 12, 4 * bench.L2_BYTES)
        for mib in sizes:
            res.setdefault((st, mib), []).append(r[f"{mib}MiB"]["gbs_device"])
        s.dispose()
        s.close()
for (st, mib), v in sorted(res.items()):
    print(f"stages={st:2d} {mib:5d} MiB: {np.median(v):8.1f} GB/s {v}", flush=True)
