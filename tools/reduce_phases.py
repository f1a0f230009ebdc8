"""block_reduce_f32 phase breakdown from the device timeline (LK_CF_TIMELINE,
lk.h words 12-15): per dispatch, span = last end - first begin, and its parts:
begin skew, begin -> first bulk copy issued, issue -> first data, the
slowest worker's arrival, and the last worker's combine."""
import sys

sys.path.insert(0, ".") if "paper_2310_01212_b200" not in sys.modules else None
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor, reduce_blocks  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
import os
acq = os.environ.get("ACQ", "1") == "1"
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway", timeline=True,
                                                      acquire_poll=acq))
n = s.num_workers
full = host.full_mask(n)
for mib in [int(x) for x in sys.argv[1:]] or [4, 16, 64, 256]:
    el = (mib << 20) // 4
    nsets = max(2, min(16, (512 << 20) // (4 * el)))
    works = []
    for k in range(nsets):
        x, p, t = DeviceBuffer(4 * el), DeviceBuffer(8 * reduce_blocks(el)), DeviceBuffer(8)
        w = WorkDescriptor(slot=100 + k, kind="block_reduce_f32", data_in_ref=x, data_out_ref=p, total_ref=t)
        s.register(w, full)
        works.append((w, x, p, t))
    rows = []
    for r in range(40):
        w = works[r % nsets][0]
        s.trigger(full, w)
        s.wait(full)
        tl = s.last_timeline().astype(np.int64)
        if r < 8:
            continue
        b, e = tl[:, 1], tl[:, 2]
        last = int(np.argmax(e))
        rows.append((e.max() - b.min(), b.max() - b.min(), np.median(tl[:, 12] - b), np.median(tl[:, 14] - tl[:, 12]),
                     np.median(tl[:, 13] - tl[:, 12]), np.median(tl[:, 15] - b), (tl[:, 15] - b).max(),
                     e[last] - tl[last, 15], np.sort(tl[:, 15])[-1] - b.min()))
    a = np.median(np.array(rows, dtype=np.float64), axis=0) / 1e3
    gbs = 4 * el / (a[0] * 1e3)
    print(f"{mib:5d}MiB span {a[0]:6.2f} us ({gbs:6.0f} GB/s) | begin skew {a[1]:4.2f} | begin->issue {a[2]:4.2f} | "
          f"issue->first data {a[3]:4.2f} | issue span med {a[4]:6.2f} | arrive med {a[5]:6.2f} max {a[6]:6.2f} | "
          f"first begin->last arrival {a[8]:6.2f} | combine {a[7]:4.2f}", flush=True)
    for w, x, p, t in works:
        for bf in (x, p, t):
            bf.free()
s.dispose()
s.close()
