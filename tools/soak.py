"""Soak: one session (default config) runs mixed traffic for `minutes`
(default 5) -- round-robin and single-worker empty tasks from C, full-mask
dispatches, Python-API round robin, saxpy payloads, zero-copy vector adds
in host-mapped buffers and 16 MiB block reduces, each checked against the
oracle -- and reports any error, the rounds done and the worst latencies."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from oracle import work as W  # noqa: E402
from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, HostBuffer, WorkDescriptor, reduce_blocks  # noqa: E402

minutes = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
mode = sys.argv[2] if len(sys.argv) > 2 else "direct"
lazy = len(sys.argv) > 3 and sys.argv[3] == "lazy"
native.pin_host_thread(0)
s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN,
                                                      poll_mode=mode, lazy_ack=lazy))
n = s.num_workers
empty = WorkDescriptor(slot=0, kind="empty")
s.register(empty)
rr = [1 << i for i in range(n)]
full = host.full_mask(n)
k = 1 << 20
rng = np.random.default_rng(0)
x = rng.uniform(-1, 1, k).astype(np.float32)
y0 = rng.uniform(-1, 1, k).astype(np.float32)
dx, dy = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y0)
sax = WorkDescriptor(slot=1, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=dy, alpha=1.0)
# zero-copy: 4 workers add two host-mapped int32 arrays into a third
zn = 100_003
ha, hb, ho = HostBuffer(4 * zn), HostBuffer(4 * zn), HostBuffer(4 * zn)
zw = WorkDescriptor(slot=2, kind="vector_add_i32", data_in_ref=(ha, hb), data_out_ref=ho)
# block reduce, 16 MiB, every worker
rn = 4 << 20
xr = rng.uniform(0, 1, rn).astype(np.float32)
dxr, dpr, dtr = DeviceBuffer.from_array(xr), DeviceBuffer(8 * reduce_blocks(rn)), DeviceBuffer(8)
rw = WorkDescriptor(slot=3, kind="block_reduce_f32", data_in_ref=dxr, data_out_ref=dpr, total_ref=dtr)
r_total = np.float64(W.block_reduce_total(xr)).view(np.uint64)
rounds, worst, payloads, zero_copy, reduces = 0, 0, 0, 0, 0
deadline = time.monotonic() + 60 * minutes
while time.monotonic() < deadline:
    _, done, cyc = s.bench_roundtrip(rr, 0, 100_000)
    rounds += len(done)
    worst = max(worst, int(cyc.max()))
    _, done, cyc = s.bench_roundtrip([1, 2], 0, 20_000)
    rounds += len(done)
    _, done, cyc = s.bench_roundtrip([full], 0, 2_000)
    rounds += len(done)
    for j in range(2_000):
        m = rr[j % n]
        s.trigger(m, empty)
        s.wait(m)
    rounds += 2_000
    s.timings.clear()
    dy.upload(y0)
    s.trigger(full, sax)
    s.wait(full)
    np.testing.assert_array_equal(dy.download(np.float32, k).view(np.uint32), W.saxpy_f32(1.0, x, y0).view(np.uint32))
    payloads += 1
    a = rng.integers(-2**31, 2**31, zn, dtype=np.int64).astype(np.int32)
    b = rng.integers(-2**31, 2**31, zn, dtype=np.int64).astype(np.int32)
    ha.array(np.int32)[:] = a
    hb.array(np.int32)[:] = b
    s.trigger(0b1111, zw)
    s.wait(0b1111)
    np.testing.assert_array_equal(ho.array(np.int32), W.vector_add_i32(a, b))
    zero_copy += 1
    s.trigger(full, rw)
    s.wait(full)
    assert dtr.download(np.float64, 1).view(np.uint64)[0] == r_total
    reduces += 1
s.dispose()
s.close()
dx.free()
dy.free()
print(f"soak {minutes:.1f} min ({mode}{', lazy ack' if lazy else ''}): {rounds} handshakes, {payloads} checked saxpy dispatches, {zero_copy} checked "
      f"zero-copy vector adds, {reduces} bit-exact 16 MiB reduces, no error; "
      f"worst round-robin cycle {worst / 1e3:.1f} us", flush=True)
