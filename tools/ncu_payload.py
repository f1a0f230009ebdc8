"""ncu target: the payload work functions as ordinary launches.

The persistent kernel cannot run under ncu (ncu serialises each launch until
it completes, and a resident LK kernel completes only after the host, blocked
inside the launch, writes EXIT).  lk_work_kernel runs the SAME device work
functions (csrc/lk_kernels.cu: run_multi -> map_chunk / reduce_chunk) on a
148-CTA grid of 512 threads -- the persistent kernel's geometry -- so its
counters (dram bytes, throughput, stall reasons) describe the payload path.

    python tools/ncu_payload.py [--mib 64] [--reps 5]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2310_01212_b200 import native  # noqa: E402
from paper_2310_01212_b200.device import BYTES_PER_ELEMENT, DeviceBuffer, WorkDescriptor, reduce_blocks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kinds", nargs="+", default=["saxpy_f32", "block_reduce_f32", "vector_add_i32"])
    args = ap.parse_args()
    n = (args.mib << 20) // 4
    base = native.LaunchSyncBaseline(device=0)
    x, y, o = DeviceBuffer(4 * n), DeviceBuffer(4 * n), DeviceBuffer(4 * n)
    parts, tot = DeviceBuffer(8 * reduce_blocks(n)), DeviceBuffer(8)
    works = {
        "saxpy_f32": WorkDescriptor(slot=0, kind="saxpy_f32", data_in_ref=(x, y), data_out_ref=y, alpha=1.5),
        "vector_add_i32": WorkDescriptor(slot=0, kind="vector_add_i32", data_in_ref=(x, y), data_out_ref=o, n=n),
        "block_reduce_f32": WorkDescriptor(slot=0, kind="block_reduce_f32", data_in_ref=x, data_out_ref=parts,
                                           total_ref=tot),
        "hbm_stream": WorkDescriptor(slot=0, kind="hbm_stream", data_in_ref=x, data_out_ref=o, iterations=1),
    }
    for k in args.kinds:
        ms = [base.time_kernel(works[k], 1) for _ in range(args.reps)]
        best = min(ms)
        print(f"{k:18s} {args.mib} MiB  best {best * 1e3:8.2f} us  "
              f"{BYTES_PER_ELEMENT[k] * n / (best * 1e6):8.1f} GB/s (algorithmic)", flush=True)
    base.close()


if __name__ == "__main__":
    main()
