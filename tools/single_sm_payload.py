"""One worker (one SM) streaming a payload alone: configs[0]'s task (int32
vector add, 64 Ki elements = 768 KiB moved) and larger ones, vs the TMA ring
depth.  Per-SM bandwidth is bytes-in-flight bound (Little's law), so the
full-GPU-tuned 6 stages may be short for a lone SM."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
for st, tma in ((6, True), (12, True), (6, False)):
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, ring_stages=st, tma_payload=tma, tma_min_workers=1))
    out = []
    for n in (65536, 1 << 20):
        a, b, o = DeviceBuffer(4 * n), DeviceBuffer(4 * n), DeviceBuffer(4 * n)
        w = WorkDescriptor(slot=5, kind="vector_add_i32", data_in_ref=(a, b), data_out_ref=o)
        s.register(w, 1)
        for _ in range(50):
            s.trigger(1, w)
            s.wait(1)
        spans = []
        for _ in range(400):
            s.trigger(1, w)
            s.wait(1)
            bb, ee = s.last_spans()
            spans.append(int(ee[0]) - int(bb[0]))
        med = float(np.median(spans))
        out.append(f"n={n}: span {med / 1e3:.2f} us = {12 * n / med:.1f} GB/s")
        for x in (a, b, o):
            x.free()
    s.dispose()
    s.close()
    print(f"{'tma' if tma else 'lsu'} stages={st:2d}: " + " | ".join(out), flush=True)
