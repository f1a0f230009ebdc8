"""Ad-hoc GPU debug: run payload kinds repeatedly and report mismatches."""
import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import work as W
from paper_2310_01212_b200 import host, native
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor

s, _ = native.NativeSession.start(native.NativeConfig(spin_yield_threshold=200))
full = host.full_mask(s.num_workers)
def f32(n, seed): return np.random.default_rng(seed).uniform(-1, 1, n).astype(np.float32)
slot = 0
for n in [262144, 12345, 12345, 12347, 5, 13, 4 << 20, 12345]:
    for inplace in (True, False):
        for mask_name, mask in (("full", full), ("one", 1), ("four", 0b1111)):
            x, y = f32(n, 2), f32(n, 3)
            dx, dy = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y)
            do = dy if inplace else DeviceBuffer(4 * n)
            slot = (slot + 1) % 64
            s.trigger(mask, WorkDescriptor(slot=slot, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=do, alpha=1.5))
            s.wait(mask)
            got = do.download(np.float32, n)
            want = W.saxpy_f32(1.5, x, y)
            bad = np.where(got.view(np.uint32) != want.view(np.uint32))[0]
            print(f"n={n} inplace={inplace} mask={mask_name} bad={len(bad)} idx={bad[:8].tolist()} got={got[bad[:4]].tolist()} want={want[bad[:4]].tolist()} ptrs x={dx.ptr:#x} y={dy.ptr:#x} o={do.ptr:#x}", flush=True)
            yy = dy.download(np.float32, n)
            if not inplace:
                badin = np.where(yy != y)[0]
                if len(badin): print("   input y modified at", badin[:8].tolist())
# vector add with tails, in place
for n in [12345, 33]:
    a = np.random.default_rng(0).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    b = np.random.default_rng(1).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    da, db = DeviceBuffer.from_array(a), DeviceBuffer.from_array(b)
    slot = (slot + 1) % 64
    s.trigger(full, WorkDescriptor(slot=slot, kind="vector_add_i32", data_in_ref=(da, db), data_out_ref=db))
    s.wait(full)
    got = db.download(np.int32, n); want = W.vector_add_i32(a, b)
    bad = np.where(got != want)[0]
    print(f"vadd inplace n={n} bad={len(bad)} idx={bad[:8].tolist()}", flush=True)
s.dispose(); s.close()
