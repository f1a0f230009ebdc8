"""Where a trigger->FINISHED round trip goes: host and device stamps of each
worker's last dispatch, joined through a measured globaltimer/CLOCK_MONOTONIC
offset.  Medians over workers, microseconds.

    python tools/latency_breakdown.py [mode ...]
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)


def breakdown(label, rounds=20000, timeline=True, **kw):
    s, _ = native.NativeSession.start(native.NativeConfig(**{"num_workers": None, **kw}, spin_strategy=native.PURE_SPIN, timeline=timeline))
    n = s.num_workers
    s.register(WorkDescriptor(slot=0, kind="empty"))
    masks = [1 << i for i in range(n)]
    s.bench_roundtrip(masks, 0, 2000)
    _, done, _ = s.bench_roundtrip(masks, 0, rounds)
    t = s.last_timeline().astype(np.int64)
    h = s.last_host_times().astype(np.int64)
    s.dispose()
    s.close()
    off, rtt = native.clock_offset(0, 2000)
    dev = t[:, :5] - off          # device globaltimer stamps on the host clock
    ghz = np.median((t[:, 7] - t[:, 5]) / np.maximum(1, t[:, 3] - t[:, 0]))
    m = lambda x: float(np.median(x)) / 1e3  # noqa: E731
    row = {
        "done_p50": float(np.percentile(done, 50)) / 1e3,
        "host_trigger": m(h[:, 1] - h[:, 0]),
        "write->seen": m(dev[:, 0] - h[:, 1]),
        "done_p99.9": float(np.percentile(done, 99.9)) / 1e3,
        "seen->begin(cyc)": float(np.median(t[:, 6] - t[:, 5])),
        "begin->fin(cyc)": float(np.median(t[:, 7] - t[:, 6])),
        "seen->fin": m(dev[:, 3] - dev[:, 0]),
        "fin->host_seen": m(h[:, 2] - dev[:, 3]),
        "total(last)": m(h[:, 2] - h[:, 0]),
        "clock_rtt": rtt / 1e3,
    }
    if kw.get("poll_mode", "gateway") == "gateway":
        row["write->fwd"] = m(dev[:, 4] - h[:, 1])
        row["fwd->seen"] = m(dev[:, 0] - dev[:, 4])
    print(f"{label:28s} " + " ".join(f"{k}={v:.3f}" if isinstance(v, float) else f"{k}={v}" for k, v in row.items()),
          flush=True)


if __name__ == "__main__":
    breakdown("direct K=1 (clock64 only)", timeline=False, poll_mode="direct", poll_replicas=1)
    breakdown("direct K=1", poll_mode="direct", poll_replicas=1)
    breakdown("gateway K=1 (clock64 only)", timeline=False, poll_mode="gateway", poll_replicas=1)
    breakdown("gateway K=1", poll_mode="gateway", poll_replicas=1)
    breakdown("direct K=1 16w", poll_mode="direct", poll_replicas=1, num_workers=16)
    breakdown("direct K=1 1w", poll_mode="direct", poll_replicas=1, num_workers=1)
