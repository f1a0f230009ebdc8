"""block_reduce_f32 schedule A/B: static share (eighths of a fair share) x
pool claim size, set through LK_RED_SHARE8 / LK_RED_CLAIM for each session.

    python tools/reduce_sched.py "6,2" "8,1" "4,4,8" ...   (share8, claim[, ring stages])
"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402

native.pin_host_thread(0)
combos = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(6, 2), (8, 1)]
combos = [c if len(c) == 3 else (c[0], c[1], 6) for c in combos]
sizes = [16, 64, 1024]
res = {}
for trial in range(2):
    for sh, cl, stg in combos:
        os.environ["LK_RED_SHARE8"], os.environ["LK_RED_CLAIM"] = str(sh), str(cl)
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway", ring_stages=stg))
        r = bench.measure_payload(s, "block_reduce_f32", sizes, 12, 4 * bench.L2_BYTES)
        for mib in sizes:
            res.setdefault((sh, cl, stg, mib), []).append(r[f"{mib}MiB"]["gbs_device"])
        s.dispose()
        s.close()
for (sh, cl, stg, mib), v in sorted(res.items()):
    print(f"share={sh}/8 claim={cl} stages={stg:2d} {mib:5d} MiB: {np.median(v):8.1f} GB/s {v}", flush=True)
