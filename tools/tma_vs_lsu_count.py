"""TMA bulk ring vs 128-bit LSU loads as a function of how many workers
share a dispatch (each worker's chunk fixed at 256 Ki elements): a lone SM
streams faster with LSU loads, the whole GPU with the TMA ring.  Where is
the crossover?  saxpy_f32, L2-cold by rotating 8 buffer sets."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
counts = [1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 148]
res = {}
for trial in range(2):
    for tma in (True, False):
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway", tma_payload=tma, tma_min_workers=1))
        for c in counts:
            n = c * (1 << 18)
            mask = host.mask_of(range(c))
            sets = []
            for k in range(8):
                x, y = DeviceBuffer(4 * n), DeviceBuffer(4 * n)
                sets.append((x, y, WorkDescriptor(slot=10 + k, kind="saxpy_f32", data_in_ref=(x, y), data_out_ref=y,
                                                  alpha=1.5)))
                s.register(sets[-1][2], mask)
            spans = []
            for r in range(40):
                w = sets[r % 8][2]
                s.trigger(mask, w)
                s.wait(mask)
                b, e = s.last_spans()
                if r >= 8:
                    spans.append(int(e[:c].max()) - int(b[:c].min()))
            gbs = 12 * n / float(np.median(spans))
            res.setdefault((c, tma), []).append(gbs)
            for x, y, _ in sets:
                x.free()
                y.free()
        s.dispose()
        s.close()
for c in counts:
    t, l = np.median(res[(c, True)]), np.median(res[(c, False)])
    print(f"workers {c:3d}: tma {t:7.1f} GB/s ({t / c:5.1f}/SM) | lsu {l:7.1f} GB/s ({l / c:5.1f}/SM) | "
          f"{'LSU' if l > t else 'TMA'} by {abs(l / t - 1) * 100:4.1f}%", flush=True)
