"""bench.py's zero_copy extra on its own: small transfers through mapped
host buffers vs cudaMemcpy, and the full-board mailbox workaround."""
import json
import os
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2310_01212_b200 import native  # noqa: E402

native.init_device(0)
native.pin_host_thread(0)
cores = sorted(os.sched_getaffinity(0))
os.sched_setaffinity(0, {cores[-1]})
cfg = native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
print(json.dumps(bench.measure_zero_copy(cfg, 0, [4, 64, 1024, 4096, 16384, 65536], reps)))
