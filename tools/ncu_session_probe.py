"""Drive a live LK session under ncu and print progress to stderr (which
step a serialising profiler blocks, if any).

    ncu --metrics gpu__time_duration.sum python tools/ncu_session_probe.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def say(msg):
    print(f"[{time.monotonic():.3f}] {msg}", file=sys.stderr, flush=True)


def main():
    from paper_2310_01212_b200 import native
    from paper_2310_01212_b200.device import WorkDescriptor
    say(f"under_profiler={native.under_profiler()}")
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=8, host_descriptors=native.under_profiler()))
    say("started")
    s.trigger(1, WorkDescriptor(slot=0, kind="empty"))
    s.wait(1)
    say("empty round trip done")
    s.trigger(3, WorkDescriptor(slot=1, iterations=100))
    s.wait(3)
    say("busy loop done")
    s.dispose()
    say("disposed")
    s.close()
    say("closed")


if __name__ == "__main__":
    main()
