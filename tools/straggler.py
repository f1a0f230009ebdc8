"""Which workers finish last in a full-mask payload dispatch?  Per-worker
durations over repeated dispatches, correlated with SM id."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor  # noqa: E402

native.pin_host_thread(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "gateway"
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode=mode))
n = s.num_workers
full = host.full_mask(n)
el = (64 << 20) // 4
bufs = [(DeviceBuffer(4 * el), DeviceBuffer(4 * el)) for _ in range(4)]
works = [WorkDescriptor(slot=10 + k, kind="saxpy_f32", data_in_ref=(x, y), data_out_ref=y, alpha=1.0)
         for k, (x, y) in enumerate(bufs)]
durs, ends, begins = [], [], []
for r in range(44):
    w = works[r % 4]
    s.trigger(full, w)
    s.wait(full)
    b, e = s.last_spans()
    if r >= 4:
        b, e = b.astype(np.int64), e.astype(np.int64)
        durs.append(e - b)
        ends.append(e - b.min())
        begins.append(b - b.min())
smid = np.array(s.smid_map)
s.dispose()
s.close()
D = np.array(durs) / 1e3
E = np.array(ends) / 1e3
B = np.array(begins) / 1e3
med = np.median(D, axis=0)
order = np.argsort(-med)
print("per-worker median duration us: min %.2f p50 %.2f max %.2f" % (med.min(), np.median(med), med.max()))
print("slowest workers (wid:smid:us):", [(int(i), int(smid[i]), round(float(med[i]), 2)) for i in order[:10]])
print("fastest workers:", [(int(i), int(smid[i]), round(float(med[i]), 2)) for i in order[-5:]])
print("rank correlation of slowness across dispatches: %.2f" % np.mean(
    [np.corrcoef(D[k], D[k + 1])[0, 1] for k in range(len(D) - 1)]))
print("median begin offset us: p50 %.2f max %.2f; end offset max (span) p50 %.2f" % (
    np.median(B), np.median(B.max(axis=1)), np.median(E.max(axis=1))))
die = smid >= 74
print("median duration die0 %.2f die1 %.2f (smid < 74 vs >= 74)" % (np.median(med[~die]), np.median(med[die])))
