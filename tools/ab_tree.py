"""Two source trees A/B in alternating processes (same box): argv[1] is the
root whose paper_2310_01212_b200 package (with its own built liblk.so) is
imported, e.g. "." against an older commit unpacked under build/ab_old
(git archive <commit> paper_2310_01212_b200 include | tar -x -C build/ab_old,
then build it there).  Prints full-mask dispatch by poll mode, the
148-worker round robin and 64 MiB payload GB/s."""
import os
import sys

root = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else ".")
sys.path.insert(0, root)
sys.path.insert(1, os.path.abspath("."))
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import host, native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

assert native.__file__.startswith(root), native.__file__
native.init_device(0)
native.pin_host_thread(0)
os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
import bench  # noqa: E402


def q(x):
    return f"{np.percentile(x, 50)/1e3:5.2f}/{np.percentile(x, 99.9)/1e3:5.2f}"


out = []
for mode in ("direct", "gateway", "hybrid"):
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN,
                                                          poll_mode=mode))
    s.register(WorkDescriptor(slot=0, kind="empty"))
    full = host.full_mask(s.num_workers)
    s.bench_roundtrip([full], 0, 2000)
    _, d, c = s.bench_roundtrip([full], 0, 20000)
    out.append(f"{mode} full {q(d)} cyc {q(c)}")
    if mode == "direct":
        rr = [1 << i for i in range(s.num_workers)]
        _, d, c = s.bench_roundtrip(rr, 0, 100000)
        out.append(f"rr {q(d)}")
    if mode == "gateway":
        for kind in ("saxpy_f32", "block_reduce_f32"):
            r = bench.measure_payload(s, kind, [64], 16, 4 * bench.L2_BYTES)["64MiB"]
            out.append(f"{kind[:6]} {r['gbs_device']:.0f}/{r['gbs_e2e']:.0f}")
    s.dispose()
    s.close()
print(f"{sys.argv[1] if len(sys.argv) > 1 else '.'}: " + " | ".join(out), flush=True)
