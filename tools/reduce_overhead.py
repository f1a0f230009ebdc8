"""Where the block_reduce_f32 fixed cost goes: per-worker durations, begin
skew and the combiner's extra time, against hbm_stream at the same size."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor, reduce_blocks  # noqa: E402

native.pin_host_thread(0)
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway"))
n = s.num_workers
full = host.full_mask(n)
for mib in (4, 16, 64):
    el = (mib << 20) // 4
    sets = []
    for k in range(16):
        x, o, p, t = DeviceBuffer(4 * el), DeviceBuffer(4 * el), DeviceBuffer(8 * reduce_blocks(el)), DeviceBuffer(8)
        sets.append((x, o, p, t))
    for kind in ("block_reduce_f32", "hbm_stream"):
        works = []
        for k, (x, o, p, t) in enumerate(sets):
            if kind == "hbm_stream":
                w = WorkDescriptor(slot=100 + k, kind=kind, data_in_ref=x, data_out_ref=o, iterations=1)
            else:
                w = WorkDescriptor(slot=100 + k, kind=kind, data_in_ref=x, data_out_ref=p, total_ref=t)
            s.register(w, full)
            works.append(w)
        rows = []
        for r in range(40):
            s.trigger(full, works[r % 16])
            s.wait(full)
            b, e = s.last_spans()
            b, e = b.astype(np.int64), e.astype(np.int64)
            if r >= 8:
                d = e - b
                last = int(np.argmax(e))
                rows.append((e.max() - b.min(), b.max() - b.min(), np.median(d), d.max(), d[last],
                             np.sort(e)[-1] - np.sort(e)[-2]))
        a = np.median(np.array(rows, dtype=np.float64), axis=0) / 1e3
        print(f"{mib:3d}MiB {kind:17s} span {a[0]:6.2f} | skew {a[1]:5.2f} | dur med {a[2]:6.2f} max {a[3]:6.2f} "
              f"last-ender {a[4]:6.2f} | last-end gap {a[5]:5.2f} us", flush=True)
    for x, o, p, t in sets:
        for bf in (x, o, p, t):
            bf.free()
s.dispose()
s.close()
