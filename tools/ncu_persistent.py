"""The persistent kernel itself under ncu: lk_profile_run boots a DIRECT
session whose round-robin empty-task handshakes come from a host thread
started before the launch, so ncu's serialized launch returns.  Run as

    ncu --replay-mode application --clock-control none --set full \\
        -k lk_persistent_kernel -c 1 -o out python tools/ncu_persistent.py [rounds]

Without ncu it prints the rounds' tasks/s (a sanity check of the hook)."""
import sys

sys.path.insert(0, ".")
from paper_2310_01212_b200 import native  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
native.pin_host_thread(0)
ns = native.profile_run(native.NativeConfig(), rounds)
print(f"profile run: {rounds} round-robin empty tasks in {ns / 1e6:.1f} ms = {rounds / (ns / 1e9) / 1e3:.1f}k tasks/s",
      flush=True)
