"""Every NativeConfig knob that changes the device or host data path, each on
one session running the same mixed program: round-robin empty tasks, a busy
loop, overlapping dispatches on disjoint workers, full-mask saxpy_f32 and
block_reduce_f32 payloads checked against the oracle, and the whole trace
replayed by the oracle validator and checked against the golden per-worker
projection (oracle/projection.py)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import projection
from oracle import protocol as O
from oracle import work as W
from paper_2310_01212_b200 import host, native
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor, reduce_blocks
from paper_2310_01212_b200.errors import UsageError

pytestmark = pytest.mark.gpu

NW = 16

KNOBS = {
    "cell8": dict(cell_stride=8),
    "cell64": dict(cell_stride=64),
    "status16": dict(status_stride=16),
    "status128": dict(status_stride=128),
    "status32-cell16": dict(status_stride=32, cell_stride=16),
    "threads32": dict(threads_per_worker=32),           # producer and consumer in one warp
    "threads64": dict(threads_per_worker=64),
    "threads544": dict(threads_per_worker=544),
    "backoff": dict(poll_backoff_ns=400),
    "relaxed-poll": dict(acquire_poll=False),
    "fence-always": dict(fence_always=True),
    "no-ack-delay": dict(ack_delay_ns=0),
    "idle-delay": dict(idle_delay_ns=300),
    "ack-fixed": dict(ack_adaptive=False, ack_delay_ns=250),
    "ack-delay-1us": dict(ack_delay_ns=1000, idle_delay_ns=1500),
    "timeline": dict(timeline=True, poll_mode="gateway"),
    "pure-spin": dict(spin_strategy=native.PURE_SPIN),
    "stages2": dict(ring_stages=2),
    "lsu-below-17": dict(tma_min_workers=17),      # NW=16: every dispatch on LSU loads
    "stages12-lsu": dict(ring_stages=12, tma_payload=False),
    "slots8": dict(num_slots=8),
    "full-board": dict(full_board=True),
    "hybrid": dict(poll_mode="hybrid"),
}


@pytest.mark.parametrize("name", list(KNOBS))
def test_knob_program(name):
    kw = dict(KNOBS[name])
    kw.setdefault("tma_min_workers", 1)   # NW=16 workers: keep the ring path under test
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=NW, record_trace=True, trace_capacity=2048,
                                                          spin_yield_threshold=200, **kw))
    bufs = []
    try:
        program = []
        empty = WorkDescriptor(slot=0, kind="empty")
        for k in range(3 * NW):
            m = 1 << (k % NW)
            s.trigger(m, empty)
            s.wait(m)
            program.append((m, 0))
        busy = WorkDescriptor(slot=1, iterations=5000)
        s.trigger(0b11, busy)
        s.trigger(0b1100, WorkDescriptor(slot=2, kind="empty"))
        s.wait(0b1100)
        s.wait(0b11)
        program += [(0b11, 1), (0b1100, 2)]

        full = host.full_mask(NW)
        n = 300_001
        rng = np.random.default_rng(11)
        x = rng.uniform(-1, 1, n).astype(np.float32)
        y = rng.uniform(-1, 1, n).astype(np.float32)
        dx, dy = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y)
        bufs += [dx, dy]
        s.trigger(full, WorkDescriptor(slot=3, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=dy, alpha=-0.75))
        s.wait(full)
        program.append((full, 3))
        np.testing.assert_array_equal(dy.download(np.float32, n).view(np.uint32),
                                      W.saxpy_f32(-0.75, x, y).view(np.uint32))

        v = rng.integers(0, 16, n).astype(np.float32)
        dv, dp, dt = DeviceBuffer.from_array(v), DeviceBuffer(8 * reduce_blocks(n)), DeviceBuffer(8)
        bufs += [dv, dp, dt]
        for rep in range(2):   # the reduce counter re-arms
            s.trigger(full, WorkDescriptor(slot=4, kind="block_reduce_f32", data_in_ref=dv, data_out_ref=dp,
                                           total_ref=dt))
            s.wait(full)
            program.append((full, 4))
            np.testing.assert_array_equal(dp.download(np.float64, reduce_blocks(n)), W.block_reduce_partials(v))
            assert dt.download(np.float64, 1)[0] == W.block_reduce_total(v)

        if s.cfg.num_slots == 8:
            with pytest.raises(UsageError):
                s.trigger(1, WorkDescriptor(slot=8, kind="empty"))
        s.dispose()

        writes = [(r.side, r.sm_id, r.word) for r in s.recorded_trace()]
        assert O.replay(writes).violation is None
        per = projection.program_slots(program, NW)
        proj = projection.projections(writes, NW)
        for i in range(NW):
            assert proj[i] == projection.expected_projection(per[i]), i
    finally:
        s.close()
        for b in bufs:
            b.free()
