"""Payload GB/s vs size and ring depth (bench.measure_payload), to separate
pipeline fill / dispatch skew from steady-state streaming."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402

native.pin_host_thread(0)
stages = [int(x) for x in sys.argv[1:]] or [6, 12]
for st in stages:
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway", ring_stages=st))
    for kind in ("saxpy_f32", "block_reduce_f32", "hbm_stream"):
        if kind == "hbm_stream":
            continue
        r = bench.measure_payload(s, kind, [16, 64, 256, 1024], 10, 4 * bench.L2_BYTES)
        print(f"stages={st} {kind}", {k: (v["gbs_device"], v["device_span_us"]) for k, v in r.items()}, flush=True)
    s.dispose()
    s.close()
