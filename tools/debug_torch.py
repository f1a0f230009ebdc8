"""Find where torch blocks while a persistent LK kernel is resident (debug aid)."""
import faulthandler
import sys
import time
sys.path.insert(0, ".")
faulthandler.dump_traceback_later(25, exit=True)
import numpy as np
import torch
from paper_2310_01212_b200 import native
from paper_2310_01212_b200.device import WorkDescriptor


def step(msg):
    print(f"{time.monotonic():.3f} {msg}", flush=True)


torch.zeros(1, device="cuda")
torch.cuda.synchronize()
step("torch up")
s, _ = native.NativeSession.start(native.NativeConfig(spin_yield_threshold=200))
step("session up")
a = np.arange(100_000, dtype=np.int32)
t = torch.from_numpy(a)
step("from_numpy")
ta = t.cuda()
step(".cuda() done")
tb = ta + 1
step("elementwise kernel done (async)")
torch.cuda.current_stream().synchronize()
step("current_stream sync done")
to = torch.empty_like(ta)
s.trigger(0b11, WorkDescriptor(slot=60, kind="vector_add_i32", data_in_ref=(ta, tb), data_out_ref=to))
s.wait(0b11)
step("lk dispatch done")
print(to[:4].cpu(), flush=True)
step(".cpu() done")
big = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
step("new segment alloc done")
del big
torch.cuda.empty_cache()
step("empty_cache done")
s.close()
step("closed")
