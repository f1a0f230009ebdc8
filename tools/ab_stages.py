"""A/B of the TMA ring depth, interleaved trials (bench.measure_payload)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402

native.pin_host_thread(0)
stages = [int(x) for x in sys.argv[1:]] or [6, 8, 12]
res = {k: {} for k in stages}
for trial in range(3):
    for st in stages:
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway", ring_stages=st))
        for kind in ("saxpy_f32", "block_reduce_f32"):
            r = bench.measure_payload(s, kind, [64], 20, 4 * bench.L2_BYTES)
            res[st].setdefault(kind, []).append(r["64MiB"]["gbs_device"])
        s.dispose()
        s.close()
for st in stages:
    print(f"stages={st:2d}", {k: (round(float(np.median(v)), 1), v) for k, v in res[st].items()}, flush=True)
