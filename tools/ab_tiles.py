"""A/B: payload GB/s with the balanced tail (dynamic_tiles) on and off, same
box, alternating sessions (bench.measure_payload, L2-cold rotation)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402

native.pin_host_thread(0)
res = {True: {}, False: {}}
for trial in range(3):
    for dyn in (True, False):
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway", dynamic_tiles=dyn))
        r = bench.measure_payload(s, "saxpy_f32", [16, 64], 20, 4 * bench.L2_BYTES)
        s.dispose()
        s.close()
        for k, v in r.items():
            res[dyn].setdefault(k, []).append(v["gbs_device"])
for dyn in (True, False):
    print("dynamic" if dyn else "static ", {k: (round(float(np.median(v)), 1), v) for k, v in res[dyn].items()})
