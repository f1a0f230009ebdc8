"""TMA ring vs LSU loads at full width (148 workers) across sizes, saxpy_f32
and block_reduce_f32, L2-cold (rotating >= 4x L2 of buffers)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402

native.pin_host_thread(0)
res = {}
for trial in range(2):
    for path in ("ring", "lsu"):
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode="gateway", tma_payload=path == "ring"))
        for kind in ("saxpy_f32", "block_reduce_f32"):
            r = bench.measure_payload(s, kind, [16, 64, 256, 1024], 8, 4 * bench.L2_BYTES)
            for k, v in r.items():
                res.setdefault((kind, k, path), []).append(v["gbs_device"])
        s.dispose()
        s.close()
for kind in ("saxpy_f32", "block_reduce_f32"):
    for size in ("16MiB", "64MiB", "256MiB", "1024MiB"):
        a, b = max(res[(kind, size, "ring")]), max(res[(kind, size, "lsu")])
        print(f"{kind:17s} {size:8s} ring {a:7.1f} | lsu {b:7.1f} GB/s | {'LSU' if b > a else 'ring'} by "
              f"{abs(b / a - 1) * 100:4.1f}%", flush=True)
