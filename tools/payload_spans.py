"""Per-worker begin/end of one payload dispatch (globaltimer): how much of the
span is dispatch skew, how much the slowest worker's chunk."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor, reduce_blocks  # noqa: E402

native.pin_host_thread(0)
for mode in ("gateway", "direct"):
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode=mode))
    n = s.num_workers
    full = host.full_mask(n)
    el = (64 << 20) // 4
    sets = []
    for k in range(8):
        x, p, t = DeviceBuffer(4 * el), DeviceBuffer(8 * reduce_blocks(el)), DeviceBuffer(8)
        sets.append((x, p, t, WorkDescriptor(slot=10 + k, kind="block_reduce_f32", data_in_ref=x, data_out_ref=p,
                                             total_ref=t)))
        s.register(sets[-1][3], full)
    for kind in ("block_reduce_f32", "saxpy_f32"):
        spans, skews, durs = [], [], []
        for r in range(24):
            x, p, t, w = sets[r % 8]
            if kind == "saxpy_f32":
                x2 = sets[(r + 1) % 8][0]
                w = WorkDescriptor(slot=30 + r % 4, kind="saxpy_f32", data_in_ref=(x, x2), data_out_ref=x2, alpha=1.0)
            s.trigger(full, w)
            s.wait(full)
            b, e = s.last_spans()
            b, e = b.astype(np.int64), e.astype(np.int64)
            if r >= 4:
                spans.append(e.max() - b.min())
                skews.append(b.max() - b.min())
                durs.append(np.median(e - b))
        print(f"{mode:8s} {kind:17s} span {np.median(spans)/1e3:6.2f} us | begin skew {np.median(skews)/1e3:5.2f} us "
              f"| median worker duration {np.median(durs)/1e3:6.2f} us", flush=True)
    s.dispose()
    s.close()
