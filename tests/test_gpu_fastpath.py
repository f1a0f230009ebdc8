"""The kernel fast path (lk_kernels.cu: fast_step) under trace parity.

configs[1] -- the benchmarked path -- settles every handshake in fast_step:
IDLE x WORK(empty) publishes WORKING + FINISHED in place, FINISHED x NOP
publishes NOP.  With record_trace on, those publishes append the same device
trace records as the general path, so these sessions replay the fast path
itself through the ORACLE validator (oracle/protocol.py, pinned to the
reference's goldens) and the golden per-worker projection
D0 D4 (H[16+slot] D2 D1 H4 D4)* H8 (P/protocol.py:151-206, P/native.py:208-299).
lk_fast_count proves the branches ran: exactly two fast steps per dispatch.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import projection
from oracle import protocol as O
from oracle import work as W
from paper_2310_01212_b200 import host, native, protocol
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor

pytestmark = pytest.mark.gpu


def _bench_cfg(**kw):
    """bench.py's configs[1] session: DIRECT polling, one worker per SM, the
    adaptive ack delay, pure host spin -- plus the trace."""
    base = dict(num_workers=None, spin_strategy=native.PURE_SPIN, poll_mode="direct", poll_replicas=1,
                cell_stride=128, poll_backoff_ns=0, record_trace=True, trace_capacity=4096)
    base.update(kw)
    return native.NativeConfig(**base)


def _replay(session, program):
    writes = [(r.side, r.sm_id, r.word) for r in session.recorded_trace()]
    r = O.replay(writes)
    assert r.violation is None, r.violation
    assert protocol.validate_trace(writes) is None
    assert all(a == b for a, b in r.dispatch_counts().values())   # exactly once
    n = session.num_workers
    per = projection.program_slots(program, n)
    proj = projection.projections(writes, n)
    for i in range(n):
        assert proj[i] == projection.expected_projection(per[i]), i
    return writes


def test_configs1_roundrobin_fast_path_replays():
    """The bench's exact loop (lk_bench_roundtrip, round robin over every SM,
    empty task with LK_HINT_EMPTY) with the trace on."""
    s, _ = native.NativeSession.start(_bench_cfg())
    try:
        n = s.num_workers
        s.register(WorkDescriptor(slot=0, kind="empty"))
        masks = [1 << i for i in range(n)]
        rounds = 40 * n
        _, done, _ = s.bench_roundtrip(masks, 0, rounds)
        fast = s.fast_counts()
        s.dispose()
        _replay(s, [(masks[k % n], 0) for k in range(rounds)])
        # IDLE x WORK(empty) and FINISHED x NOP: two fast steps per dispatch, per worker
        np.testing.assert_array_equal(fast, np.full(n, 2 * 40, dtype=np.uint32))
        assert np.median(done) > 0
    finally:
        s.close()


def test_full_mask_fast_path_replays():
    s, _ = native.NativeSession.start(_bench_cfg())
    try:
        n = s.num_workers
        s.register(WorkDescriptor(slot=3, kind="empty"))
        full = host.full_mask(n)
        s.bench_roundtrip([full], 3, 200)
        fast = s.fast_counts()
        s.dispose()
        _replay(s, [(full, 3)] * 200)
        np.testing.assert_array_equal(fast, np.full(n, 400, dtype=np.uint32))
    finally:
        s.close()


def test_reference_default_descriptor_is_fast():
    """busy_loop(0) -- the reference's WorkDescriptor(slot) default
    (P/device.py:48-66) -- rides the empty-task fast path through the Python API."""
    s, _ = native.NativeSession.start(_bench_cfg(num_workers=8))
    try:
        w = WorkDescriptor(slot=5)
        program = []
        for k in range(64):
            m = 1 << (k % 8)
            s.trigger(m, w)
            s.wait(m)
            program.append((m, 5))
        fast = s.fast_counts()
        s.dispose()
        _replay(s, program)
        np.testing.assert_array_equal(fast, np.full(8, 16, dtype=np.uint32))
    finally:
        s.close()


def test_cached_busy_loop_fast_path_replays():
    """Re-dispatching a staged busy_loop: the first dispatch to a worker
    fetches the descriptor (general path), every later one carries
    LK_HINT_CACHED and runs the loop inside fast_step."""
    nw = 16
    s, _ = native.NativeSession.start(_bench_cfg(num_workers=nw))
    try:
        w = WorkDescriptor(slot=7, iterations=64)
        program = []
        for k in range(10 * nw):
            m = 1 << (k % nw)
            s.trigger(m, w)
            s.wait(m)
            program.append((m, 7))
        fast = s.fast_counts()
        s.dispose()
        _replay(s, program)
        # per worker: 10 acks (FINISHED x NOP) + 10 begins: the first fetches the
        # descriptor (fast begin, loop in the general path), 9 run cached in place
        np.testing.assert_array_equal(fast, np.full(nw, 2 * 10, dtype=np.uint32))
    finally:
        s.close()


def test_cached_saxpy_redispatch_fast_begin():
    """A payload slot re-triggered on the same mask: IDLE x WORK begins in
    fast_step from the cached descriptor, results bit-exact each time."""
    nw = 32
    s, _ = native.NativeSession.start(_bench_cfg(num_workers=nw))
    bufs = []
    try:
        n = 100_003
        x = np.random.default_rng(2).uniform(-1, 1, n).astype(np.float32)
        y = np.random.default_rng(3).uniform(-1, 1, n).astype(np.float32)
        dx, dy = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y)
        bufs += [dx, dy]
        full = host.full_mask(nw)
        w = WorkDescriptor(slot=9, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=dy, alpha=1.5)
        want = y
        reps = 12
        for _ in range(reps):
            s.trigger(full, w)
            s.wait(full)
            want = W.saxpy_f32(1.5, x, want)
            np.testing.assert_array_equal(dy.download(np.float32, n).view(np.uint32), want.view(np.uint32))
        fast = s.fast_counts()
        s.dispose()
        _replay(s, [(full, 9)] * reps)
        # every dispatch begins in fast_step (payload kinds never skip it) + every ack
        np.testing.assert_array_equal(fast, np.full(nw, 2 * reps, dtype=np.uint32))
    finally:
        s.close()
        for b in bufs:
            b.free()


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_mixed_program_fast_and_general_paths(seed):
    """Random interleavings of empty, cached busy loops, payloads, partial
    waits and re-staged slots, so fast-path and general-path steps alternate
    on the same workers; every trace replays."""
    import random
    rng = random.Random(seed)
    nw = 24
    s, _ = native.NativeSession.start(_bench_cfg(num_workers=nw, lazy_ack=rng.random() < 0.5))
    nrng = np.random.default_rng(seed)
    bufs = []
    try:
        n = 4096
        x = nrng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
        dx, do = DeviceBuffer.from_array(x), DeviceBuffer(4 * n)
        bufs += [dx, do]
        works = [WorkDescriptor(slot=0, kind="empty"), WorkDescriptor(slot=1, iterations=16),
                 WorkDescriptor(slot=2, iterations=0),
                 WorkDescriptor(slot=3, kind="vector_add_i32", data_in_ref=(dx, dx), data_out_ref=do)]
        program = []
        for step in range(150):
            w = rng.choice(works)
            if w.slot == 3:
                mask = host.full_mask(nw)
            else:
                ids = rng.sample(range(nw), rng.randint(1, 4))
                mask = host.mask_of(ids)
            if rng.random() < 0.05:   # re-stage: a fresh object for the slot invalidates worker caches
                w = WorkDescriptor(slot=1, iterations=rng.randrange(1, 40))
                works[1] = w
            s.trigger(mask, w)
            program.append((mask, w.slot))
            s.wait(mask)
            if w.slot == 3:
                np.testing.assert_array_equal(do.download(np.int32, n), W.vector_add_i32(x, x))
        fast = s.fast_counts()
        s.dispose()
        _replay(s, program)
        assert fast.sum() > len(program)   # the fast path carried most steps
    finally:
        s.close()
        for b in bufs:
            b.free()


def test_roundtrip_gaps_probe():
    """lk_bench_roundtrip_gaps runs the same handshakes (trace replays) and
    reports a host spin gap per round."""
    s, _ = native.NativeSession.start(_bench_cfg(num_workers=16))
    try:
        s.register(WorkDescriptor(slot=0, kind="empty"))
        masks = [1 << i for i in range(16)]
        _, done, cyc, gap = s.bench_roundtrip_gaps(masks, 0, 320)
        assert gap.shape == done.shape and (cyc >= done).all()
        assert np.median(gap) < np.median(cyc)   # a typical round is not one long stall
        s.dispose()
        _replay(s, [(masks[k % 16], 0) for k in range(320)])
    finally:
        s.close()
