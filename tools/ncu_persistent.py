"""The persistent kernel itself under ncu: lk_profile_run boots a DIRECT
session whose dispatches come from a host thread started before the launch,
so ncu's serialized launch returns.  Run as

    ncu --replay-mode application --clock-control none --set full \\
        -k lk_persistent_kernel -c 1 -o out python tools/ncu_persistent.py [rounds] [saxpy]

No second argument: round-robin empty tasks (configs[1] shape).  `saxpy`:
full-mask saxpy_f32 dispatches, 64 MiB per vector, rotating over 4 buffer
sets (512 MiB, L2-cold), for the in-situ DRAM traffic per dispatch.
`reduce`: full-mask block_reduce_f32 over 64 MiB, rotating 8 buffers.
Without ncu it prints the run's rate (a sanity check of the hook)."""
import sys

sys.path.insert(0, ".")
from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor, reduce_blocks  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
kind = sys.argv[2] if len(sys.argv) > 2 else ""
payload = kind in ("saxpy", "reduce")
native.pin_host_thread(0)
if not payload:
    ns = native.profile_run(native.NativeConfig(num_workers=None), rounds)
    print(f"profile run: {rounds} round-robin empty tasks in {ns / 1e6:.1f} ms = "
          f"{rounds / (ns / 1e9) / 1e3:.1f}k tasks/s", flush=True)
else:
    n = (64 << 20) // 4
    bufs, works = [], []
    for k in range(4 if kind == "saxpy" else 8):
        if kind == "saxpy":
            x, y = DeviceBuffer(4 * n), DeviceBuffer(4 * n)
            bufs += [x, y]
            works.append(WorkDescriptor(slot=1 + k, kind="saxpy_f32", data_in_ref=(x, y), data_out_ref=y, alpha=1.5))
        else:
            x, part, tot = DeviceBuffer(4 * n), DeviceBuffer(8 * reduce_blocks(n)), DeviceBuffer(8)
            bufs += [x, part, tot]
            works.append(WorkDescriptor(slot=1 + k, kind="block_reduce_f32", data_in_ref=x, data_out_ref=part,
                                        total_ref=tot))
    ns = native.profile_run(native.NativeConfig(num_workers=None), rounds, works)
    alg = (12 if kind == "saxpy" else 4) * n
    print(f"profile run: {rounds} full-mask {works[0].kind} dispatches (64 MiB/vector) in {ns / 1e6:.2f} ms = "
          f"{rounds * alg / ns:.1f} GB/s including handshakes; algorithmic bytes/dispatch {alg}", flush=True)
    for b in bufs:
        b.free()
