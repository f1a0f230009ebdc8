"""configs[3] interference test on each poll mode (bench.measure_interference)."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402

native.pin_host_thread(0)
for mode in sys.argv[1:] or ["direct", "hybrid", "gateway"]:
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, poll_mode=mode))
    r = bench.measure_interference(s, 16, 50000, 512)
    s.dispose()
    s.close()
    print(mode, json.dumps({k: r[k] for k in ("solo", "co_running", "stream_gbs_host", "stream_gbs_device_last",
                                                "stream_dispatches")}), flush=True)
