"""Where the ack half of an empty-task cycle goes (DIRECT session, timeline
on): device FINISHED issue -> host sees it -> host writes NOP -> device sees
it (and how many cell loads that took) -> host sees NOP.  Device globaltimer
stamps are put on the host clock with lk_clock_offset.  Medians over the
last dispatch of each of the 148 workers, microseconds."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import WorkDescriptor  # noqa: E402

native.pin_host_thread(0)


def run(label, rounds=14800, **kw):
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_strategy=native.PURE_SPIN, timeline=True, **kw))
    n = s.num_workers
    s.register(WorkDescriptor(slot=0, kind="empty"))
    masks = [1 << i for i in range(n)]
    s.bench_roundtrip(masks, 0, 2000)
    _, done, cyc = s.bench_roundtrip(masks, 0, rounds)
    t = s.last_timeline().astype(np.int64)
    h = s.last_host_times().astype(np.int64)
    s.dispose()
    s.close()
    off, rtt = native.clock_offset(0, 2000)
    last = cyc[rounds - n:].astype(np.int64)            # worker i's last round is rounds - n + i
    h_nop = h[:, 0] + last
    m = lambda x: float(np.median(x)) / 1e3  # noqa: E731
    row = {
        "WORK write->dev seen": m(t[:, 0] - off - h[:, 1]),
        "dev seen->FIN issue": m(t[:, 8] - t[:, 0]),
        "FIN issue->host seen": m(h[:, 2] - (t[:, 8] - off)),
        "host FIN seen->dev NOP seen": m(t[:, 9] - off - h[:, 2]),
        "loads": float(np.median(t[:, 10])),
        "dev NOP seen->host NOP seen": m(h_nop - (t[:, 9] - off)),
        "cycle": m(last),
        "echo rtt": rtt / 1e3,
    }
    print(f"{label:10s} " + " | ".join(f"{k} {v:.3f}" for k, v in row.items()), flush=True)


for trial in range(2):
    run("no-delay", ack_delay_ns=0)
    run("delay200")
    run("delay400", ack_delay_ns=400)
