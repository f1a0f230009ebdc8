"""A short LK session for compute-sanitizer (one tool per run): boot, empty
and busy tasks, every payload kind on a few workers, trace on, dispose."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "direct"
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=8, record_trace=True, trace_capacity=256,
                                                      poll_mode=mode, wait_timeout_s=60))
n = 4096 + 7
a = np.arange(n, dtype=np.int32)
da, db, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(a), DeviceBuffer(4 * n)
p, t = DeviceBuffer(4 * 8), DeviceBuffer(8)
works = [WorkDescriptor(slot=0, kind="empty"), WorkDescriptor(slot=1, iterations=100),
         WorkDescriptor(slot=2, kind="vector_add_i32", data_in_ref=(da, db), data_out_ref=do),
         WorkDescriptor(slot=3, kind="saxpy_f32", data_in_ref=(da, db), data_out_ref=do, n=n),
         WorkDescriptor(slot=4, kind="block_reduce_f32", data_in_ref=da, data_out_ref=p, total_ref=t),
         WorkDescriptor(slot=5, kind="hbm_stream", data_in_ref=da, data_out_ref=do, iterations=2)]
for k, w in enumerate(works * 2):
    m = (1 << (k % 8)) if k % 2 else 0xFF
    s.trigger(m, w)
    s.wait(m)
s.dispose()
print("records", len(s.recorded_trace()))
s.close()
print("sanitize run ok")
