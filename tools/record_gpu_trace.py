"""Record a device trace on the B200 (criterion-8 style round robin plus
mixed full-mask and payload dispatches) and write it in the reference's trace
file format (P/protocol.py:401-432) for tests/golden/."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native, protocol  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gpu_trace.txt"
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, record_trace=True, trace_capacity=512))
n = s.num_workers
x = DeviceBuffer.from_array(np.arange(1 << 16, dtype=np.float32))
y = DeviceBuffer(4 << 16)
program = []
for k in range(1500):
    if k % 100 == 99:
        m = host.full_mask(n)
        w = WorkDescriptor(slot=1, kind="saxpy_f32", data_in_ref=(x, y), data_out_ref=y, alpha=1.0)
    else:
        m = 1 << (k % n)
        w = WorkDescriptor(slot=0, iterations=k % 7)
    s.trigger(m, w)
    s.wait(m)
    program.append((m, w.slot))
s.dispose()
recs = s.recorded_trace()
s.close()
with open(out, "w") as f:
    f.write(protocol.format_trace(recs))
print(f"{len(recs)} records, {n} workers -> {out}")
