"""Payload GB/s in the persistent kernel vs TMA ring depth (and the LSU path),
L2-cold by buffer rotation (bench.measure_payload)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402

native.pin_host_thread(0)
for tma, stages in ((False, 12), (True, 4), (True, 6), (True, 8), (True, 12)):
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway", tma_payload=tma, ring_stages=stages))
    out = {}
    for kind in ("saxpy_f32", "block_reduce_f32"):
        r = bench.measure_payload(s, kind, [4, 64], 20, 4 * bench.L2_BYTES)
        out[kind] = {k: v["gbs_device"] for k, v in r.items()}
    s.dispose()
    s.close()
    print(f"{'tma' if tma else 'lsu'} stages={stages:2d}: {out}", flush=True)
