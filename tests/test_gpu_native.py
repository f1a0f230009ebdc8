"""The reference's native-executor suite (/root/reference/pkg/tests/test_native.py)
run against the B200 session, plus GPU-only protocol parity checks.

Every trace is validated by the ORACLE replay (oracle/protocol.py, pinned to
the reference's golden vectors) and by the product's native validator, and
each worker's projection must equal the reference's golden form
D0 D4 (H[16+slot] D2 D1 H4 D4)* H8.
"""
from __future__ import annotations

import random
import statistics

import numpy as np
import pytest

from oracle import projection
from oracle import protocol as O
from paper_2310_01212_b200 import _lib, host, native, protocol
from paper_2310_01212_b200.device import WorkDescriptor
from paper_2310_01212_b200.errors import (BusyTriggerError, DisposeWhileBusyError, HangDetected,
                                          UsageError)

pytestmark = pytest.mark.gpu

FAST = dict(spin_yield_threshold=200, record_trace=True)
TINY_WORK = WorkDescriptor(slot=0, iterations=32)


_LIVE: list = []


@pytest.fixture(autouse=True)
def _reclaim_gpu():
    """A test that leaves a session resident (dead worker, failed assert) must
    not starve the next one of SMs: abort whatever is still running."""
    yield
    while _LIVE:
        s = _LIVE.pop()
        s.close()


def start(num_workers=4, **kw):
    cfg = native.NativeConfig(num_workers=num_workers, **{**FAST, **kw})
    session, _ = native.NativeSession.start(cfg)
    _LIVE.append(session)
    return session


def writes_of(session):
    return [(r.side, r.sm_id, r.word) for r in session.recorded_trace()]


def assert_trace_ok(session, program=None, num_workers=None):
    w = writes_of(session)
    r = O.replay(w)
    assert r.violation is None, r.violation
    v = protocol.validate_trace(w)
    assert v is None, v
    assert all(a == b for a, b in r.dispatch_counts().values())   # exactly once
    if program is not None:
        per = projection.program_slots(program, num_workers)
        proj = projection.projections(w, num_workers)
        for i in range(num_workers):
            assert proj[i] == projection.expected_projection(per[i]), i
    return r


# ------------------------------------------------ reference test_native.py, one for one

def test_start_brings_workers_to_idle():
    session = start(4)
    assert session.from_gpu == [protocol.NOP] * 4
    assert all(p is protocol.Phase.IDLE for p in session.worker_phase)
    session.dispose()


def test_minimal_single_worker_session():
    session = start(1)
    assert session.from_gpu == [protocol.NOP]
    session.trigger(1, TINY_WORK)
    session.wait(1)
    session.dispose()


def test_boot_is_announced_in_the_trace():
    session = start(2)
    session.dispose()
    for worker in (0, 1):
        words = [r.word for r in session.recorded_trace()
                 if r.side == protocol.DEVICE_SIDE and r.sm_id == worker]
        assert words[:2] == [protocol.INIT, protocol.NOP]


def test_zero_iteration_roundtrip_validates():
    session = start(2)
    session.trigger(0b01, WorkDescriptor(slot=0, iterations=0))
    session.wait(0b01)
    session.dispose()
    assert_trace_ok(session, [(0b01, 0)], 2)


def test_multi_worker_stress_smoke():
    session = start(4)
    cycles = 400
    for k in range(cycles):
        mask = 1 << (k % 4)
        session.trigger(mask, TINY_WORK)
        session.wait(mask)
    session.dispose()
    r = assert_trace_ok(session, [(1 << (k % 4), 0) for k in range(cycles)], 4)
    assert sum(w for w, _ in r.dispatch_counts().values()) == cycles


def test_full_mask_dispatch():
    session = start(4)
    session.trigger(0b1111, TINY_WORK)
    session.wait(0b1111)
    session.dispose()
    assert_trace_ok(session, [(0b1111, 0)], 4)


def test_single_writer_word_sets():
    session = start(2)
    session.trigger(0b11, TINY_WORK)
    session.wait(0b11)
    session.dispose()
    for rec in session.recorded_trace():
        if rec.side == protocol.HOST_SIDE:
            assert rec.word in (protocol.NOP, protocol.EXIT) or rec.word >= protocol.WORK_BASE
        else:
            assert rec.word in protocol.FROM_GPU_WORDS


def test_retrigger_busy_worker_rejected():
    session = start(2)
    session.trigger(0b01, WorkDescriptor(slot=0, iterations=200_000))
    with pytest.raises(BusyTriggerError):
        session.trigger(0b01, TINY_WORK)
    session.wait(0b01)
    session.dispose()


def test_dispose_joins_every_thread():
    session = start(4)
    session.trigger(0b1111, TINY_WORK)
    session.wait(0b1111)
    session.dispose()
    assert all(not th.is_alive() for th in session._threads)
    with pytest.raises(UsageError):
        session.trigger(1, TINY_WORK)


def test_dispose_while_pending_rejected():
    session = start(2)
    session.trigger(0b10, TINY_WORK)
    with pytest.raises(DisposeWhileBusyError):
        session.dispose()
    session.wait(0b10)
    session.dispose()


def test_spin_until_times_out():
    session = start(1, wait_timeout_s=0.05)
    with pytest.raises(HangDetected):
        session._spin_until(lambda: False, "test condition", [0])
    session.dispose()


def test_trigger_latency_beats_kernel_launch():
    session = start(4)
    work = WorkDescriptor(slot=0, iterations=64)
    trigger_ns = []
    for k in range(300):
        mask = 1 << (k % 4)
        trigger_ns.append(session.trigger(mask, work).cycles)
        session.wait(mask)
    session.dispose()
    baseline = native.LaunchSyncBaseline(grid=1)
    spawn_ns = []
    for _ in range(300):
        spawn_ns.append(baseline.launch(work).cycles)
        baseline.wait()
    baseline.close()
    assert statistics.median(trigger_ns) < statistics.median(spawn_ns)


def test_descriptor_slot_locked_while_in_flight():
    session = start(2)
    session.trigger(0b01, WorkDescriptor(slot=0, iterations=100_000))
    with pytest.raises(UsageError):
        session.trigger(0b10, WorkDescriptor(slot=0, iterations=10))
    session.trigger(0b10, WorkDescriptor(slot=1, iterations=10))
    session.wait(0b11)
    session.trigger(0b01, TINY_WORK)
    session.wait(0b01)
    session.dispose()
    assert_trace_ok(session)


def test_timing_rows_carry_backend_column():
    session = start(1)
    t = session.trigger(1, TINY_WORK)
    session.wait(1)
    session.dispose()
    text = host.timings_csv([("r0", host.MODEL_LK, t)], backend=native.BACKEND)
    assert text.splitlines()[1] == f"r0,LK,Trigger,1,{t.cycles},b200"


def test_pinning_request_downgrades_gracefully():
    session = start(2, pin_to_cores=True)
    session.trigger(0b11, TINY_WORK)
    session.wait(0b11)
    session.dispose()


def test_config_validation():
    with pytest.raises(UsageError):
        native.NativeConfig(num_workers=0)
    with pytest.raises(UsageError):
        native.NativeConfig(spin_strategy="nap")
    with pytest.raises(UsageError):
        native.NativeConfig(spin_strategy=native.SPIN_THEN_YIELD, spin_yield_threshold=0)


def test_pure_spin_roundtrip():
    session = start(1, spin_strategy=native.PURE_SPIN)
    session.trigger(1, TINY_WORK)
    session.wait(1)
    session.dispose()
    assert_trace_ok(session, [(1, 0)], 1)


# ------------------------------------------------ B200-specific

def test_all_sms_one_worker_each():
    session = start(None, record_trace=False)
    n = session.num_workers
    assert n == 148
    smids = session.smid_map
    assert len(set(smids)) == n                 # one CTA per SM, all distinct
    full = host.full_mask(n)
    session.trigger(full, WorkDescriptor(slot=0, kind="empty"))
    session.wait(full)
    session.dispose()


def test_full_gpu_trace_and_wide_masks():
    session = start(None, trace_capacity=4096)
    n = session.num_workers
    full = host.full_mask(n)
    prog = [(full, 0), (1 << (n - 1), 1), ((1 << 64) | (1 << 128) | 1, 2), (full, 3)]
    for mask, slot in prog:
        session.trigger(mask, WorkDescriptor(slot=slot, kind="empty"))
        session.wait(mask)
    with pytest.raises(UsageError):
        session.trigger(1 << n, TINY_WORK)        # wider than the board
    with pytest.raises(UsageError):
        session.trigger(0, TINY_WORK)
    session.dispose()
    assert_trace_ok(session, prog, n)


def test_wait_on_untriggered_worker_rejected():
    session = start(2)
    with pytest.raises(UsageError):
        session.wait(0b01)
    session.trigger(0b01, TINY_WORK)
    with pytest.raises(UsageError):
        session.wait(0b11)
    session.wait(0b01)
    session.dispose()


def test_partial_wait_frees_slot_only_when_all_bits_waited():
    session = start(4)
    session.trigger(0b0011, WorkDescriptor(slot=3, iterations=10))
    session.wait(0b0001)
    with pytest.raises(UsageError):
        session.trigger(0b0100, WorkDescriptor(slot=3, iterations=10))
    session.wait(0b0010)
    session.trigger(0b0100, WorkDescriptor(slot=3, iterations=10))
    session.wait(0b0100)
    session.dispose()
    assert_trace_ok(session)


def test_criterion_7_random_programs_on_gpu():
    """Random split-mask programs (T/test_acceptance.py:122-145 shape) on the device."""
    rng = random.Random(20250808)
    session = start(8, trace_capacity=4096)
    program = []
    slot = 0
    for _ in range(60):
        sms = rng.sample(range(8), rng.randint(1, 8))
        split = rng.randrange(len(sms)) if len(sms) > 1 and rng.random() < 0.3 else 0
        covered = 0
        for group in [g for g in (sms[:split], sms[split:]) if g]:
            m = host.mask_of(group)
            session.trigger(m, WorkDescriptor(slot=slot % 64, iterations=rng.randrange(400)))
            program.append((m, slot % 64))
            slot += 1
            covered |= m
        session.wait(covered)
    session.dispose()
    assert_trace_ok(session, program, 8)


@pytest.mark.parametrize("mode,seed", [("direct", 1), ("direct", 4), ("gateway", 1), ("gateway", 4),
                                       ("hybrid", 1), ("hybrid", 2)])
def test_poll_modes_random_programs(mode, seed):
    """Every to_gpu delivery path (direct PCIe polling, gateway warp + device
    mailboxes, hybrid) runs the same random programs with validated traces
    and golden projections."""
    rng = random.Random(7 + seed)
    session = start(12, trace_capacity=4096, poll_mode=mode)
    program = []
    for k in range(80):
        sms = rng.sample(range(12), rng.randint(1, 12))
        m = host.mask_of(sms)
        session.trigger(m, WorkDescriptor(slot=k % 16, iterations=rng.randrange(200)))
        program.append((m, k % 16))
        session.wait(m)
    session.dispose()
    assert_trace_ok(session, program, 12)


@pytest.mark.parametrize("mode", ["gateway", "hybrid"])
def test_gateway_back_to_back_single_worker_triggers(mode):
    """148 separate trigger events queued before any wait, then one ack event
    for the whole mask: the event ring carries them all in order."""
    session = start(None, trace_capacity=256, poll_mode=mode)
    n = session.num_workers
    work = WorkDescriptor(slot=0, kind="empty")
    for rep in range(3):
        for i in range(n):
            session.trigger(1 << i, WorkDescriptor(slot=1 + i + 150 * (rep % 2), iterations=i % 7))
        session.wait((1 << n) - 1)
    session.trigger(1, work)
    session.wait(1)
    session.dispose()
    assert_trace_ok(session)


@pytest.mark.parametrize("mode", ["direct", "gateway", "hybrid"])
def test_device_timeline_is_ordered(mode):
    session = start(None, timeline=True, poll_mode=mode)
    n = session.num_workers
    session.register(WorkDescriptor(slot=0, kind="empty"))
    session.bench_roundtrip([1 << i for i in range(n)], 0, 2 * n)
    t = session.last_timeline().astype(np.int64)
    h = session.last_host_times().astype(np.int64)
    session.dispose()
    assert (t[:, 0] > 0).all()
    assert (np.diff(t[:, :4], axis=1) >= 0).all()   # seen <= begin <= end <= finished
    if mode == "gateway":
        assert (t[:, 4] > 0).all() and (t[:, 4] <= t[:, 0]).all()   # forwarded before seen
    assert (np.diff(t[:, 5:8], axis=1) >= 0).all()  # clock64: seen <= begin <= finished
    assert np.median(t[:, 3] - t[:, 0]) < 20_000     # device-side handling well under 20 us
    assert (np.diff(h, axis=1) >= 0).all()           # host: trigger <= written <= FINISHED seen


@pytest.mark.slow
def test_criterion_8_gpu_stress():
    """10,000 round-robin cycles, zero violations, exactly-once (T/test_acceptance.py:187-223)."""
    session = start(4, trace_capacity=32768)
    work = WorkDescriptor(slot=0, iterations=32)
    trig = []
    for k in range(10_000):
        mask = 1 << (k % 4)
        trig.append(session.trigger(mask, work).cycles)
        session.wait(mask)
    session.dispose()
    r = assert_trace_ok(session, [(1 << (k % 4), 0) for k in range(10_000)], 4)
    assert sum(w for w, _ in r.dispatch_counts().values()) == 10_000


def test_c_side_roundtrip_loop_traces_validate():
    session = start(None, trace_capacity=8192)
    n = session.num_workers
    session.register(WorkDescriptor(slot=0, kind="empty"))
    masks = [1 << i for i in range(n)]
    trig, done, cyc = session.bench_roundtrip(masks, 0, 5 * n)
    assert (done > 0).all() and (cyc >= done).all()
    session.dispose()
    assert_trace_ok(session, [(masks[k % n], 0) for k in range(5 * n)], n)


def test_unregistered_slot_refused():
    session = start(1)
    rc = session._lib.lk_trigger(session._h, session._mask(1), session.nwords, 9, None, None)
    assert rc == _lib.LK_E_USAGE
    session.dispose()


@pytest.mark.parametrize("word,code", [(9, 1), (3, 1)])
def test_device_violation_surfaces_as_worker_died(word, code):
    """Fault injection: an illegal to_gpu word makes the worker record the
    violation and leave its loop; the host's next call raises (native.py:128-131)."""
    session = start(2)
    _lib.check(session._lib.lk_debug_poke(session._h, 1, word))
    session._spin_until(lambda: session.worker_phase[1] is protocol.Phase.EXITED, "device exit", [1])
    err = session.worker_error[1]
    assert err is not None and err.word == word
    with pytest.raises(UsageError, match="worker 1 died"):
        session.trigger(0b01, TINY_WORK)


def test_conflicting_slot_while_working_is_a_device_violation():
    session = start(1)
    session.trigger(1, WorkDescriptor(slot=0, iterations=2_000_000))
    _lib.check(session._lib.lk_debug_poke(session._h, 0, protocol.WORK_BASE + 5))
    session._spin_until(lambda: session.worker_phase[0] is protocol.Phase.EXITED, "device exit", [0])
    assert session.worker_error[0].word == protocol.WORK_BASE + 5


def test_baseline_launch_wait_contract():
    b = native.LaunchSyncBaseline()
    with pytest.raises(UsageError):
        b.wait()
    b.launch(WorkDescriptor(slot=0, kind="empty"))
    with pytest.raises(UsageError):
        b.launch(WorkDescriptor(slot=0, kind="empty"))
    b.wait()
    b.close()


def test_pingpong_floor_runs():
    rt = native.pingpong(0, 200)
    assert (rt > 0).all()


def test_scenario_backend_rows():
    """backend.run_b200 on a Scenario-shaped object (P/bench.py:51-116): the
    rows _run_native_lk/_run_native_baseline produce, plus the baseline's
    Dispose row the reference's native runner omits."""
    from paper_2310_01212_b200 import backend

    class Scn:
        reps = 20
        def cluster_count(self):
            return 4
        def mask(self):
            return 0b1111
        def work(self):
            return WorkDescriptor(slot=0, iterations=64)
        def models(self):
            return [host.MODEL_LK, host.MODEL_BASELINE]

    rows = backend.run_b200(Scn())
    got = {(r.model, r.phase): r for r in rows}
    for key in [("LK", "Init"), ("LK", "Trigger"), ("LK", "Wait"), ("LK", "Dispose"),
                ("BASE", "Alloc"), ("BASE", "Launch"), ("BASE", "Wait"), ("BASE", "Dispose")]:
        assert key in got, key
    assert got[("LK", "Trigger")].samples == 20 and got[("BASE", "Launch")].samples == 20
    assert all(r.best <= r.avg <= r.worst for r in rows)
    assert "b200" in backend.rows_csv(rows)


def test_hybrid_mixes_channels_per_worker():
    """HYBRID: single-worker writes take the direct cell, wide ones the ring;
    a worker alternating between both keeps one ordered write stream (the
    golden projection and the replay both hold)."""
    session = start(12, trace_capacity=4096, poll_mode="hybrid")
    full = (1 << 12) - 1
    program = []
    for k in range(40):
        if k % 3 == 0:
            m = full                          # ring event (12 > LK_HYBRID_DIRECT_MAX)
        elif k % 3 == 1:
            m = 1 << (k % 12)                 # direct cell
        else:
            m = 0b101                         # direct cells (2 workers)
        session.trigger(m, WorkDescriptor(slot=k % 8, iterations=k % 5))
        program.append((m, k % 8))
        session.wait(m)
    session.dispose()
    assert_trace_ok(session, program, 12)


def test_busy_loop_really_counts():
    """busy_loop(n) executes n iterations (native.py:63-67): the device cycles
    between work begin and FINISHED grow with n, at least one per iteration."""
    session = start(1)
    cyc = {}
    for n in (0, 100_000, 1_000_000):
        session.trigger(1, WorkDescriptor(slot=3, iterations=n))
        session.wait(1)
        t = session.last_timeline().astype(np.int64)
        cyc[n] = int(t[0, 7] - t[0, 6])
    session.dispose()
    assert cyc[1_000_000] >= 1_000_000 and cyc[100_000] >= 100_000, cyc
    assert cyc[1_000_000] > 5 * cyc[100_000] > 5 * cyc[0], cyc


@pytest.mark.parametrize("mode", ["direct", "hybrid"])
def test_lazy_ack_keeps_the_protocol(mode):
    """lazy_ack: wait() returns once the ack is written; the next trigger of
    that worker waits for the republished NOP.  Every trace still validates
    and projects to D0 D4 (H[16+slot] D2 D1 H4 D4)* H8."""
    rng = random.Random(5)
    session = start(6, trace_capacity=4096, poll_mode=mode, lazy_ack=True)
    program = []
    for k in range(120):
        m = host.mask_of(rng.sample(range(6), rng.randint(1, 6)))
        session.trigger(m, WorkDescriptor(slot=k % 4, iterations=rng.randrange(50)))
        program.append((m, k % 4))
        session.wait(m)
    session.dispose()
    assert_trace_ok(session, program, 6)


def test_lazy_ack_c_loop_roundtrips():
    session = start(None, trace_capacity=2048, lazy_ack=True)
    n = session.num_workers
    session.register(WorkDescriptor(slot=0, kind="empty"))
    masks = [1 << i for i in range(n)]
    _, done, cyc = session.bench_roundtrip(masks, 0, 4 * n)
    assert (cyc >= done).all()
    session.dispose()
    assert_trace_ok(session, [(masks[k % n], 0) for k in range(4 * n)], n)


def test_sm_partition_session():
    """sm_partition: the persistent kernel runs in a green context of 16 SMs,
    one worker per partition SM, and keeps the full protocol."""
    session = start(None, trace_capacity=2048, sm_partition=16)
    lk_sms, rest = session.partition_info
    assert session.num_workers == lk_sms >= 16 and rest > 0
    assert len(set(session.smid_map)) == session.num_workers
    rng = random.Random(3)
    program = []
    for k in range(60):
        m = host.mask_of(rng.sample(range(session.num_workers), rng.randint(1, 4)))
        session.trigger(m, WorkDescriptor(slot=k % 8, iterations=rng.randrange(100)))
        program.append((m, k % 8))
        session.wait(m)
    session.dispose()
    assert_trace_ok(session, program, session.num_workers)


def test_second_live_session_on_a_device_is_refused():
    """A live session holds every SM; a second one on the same device could
    never become resident, so start() refuses it -- and succeeds again once
    the first is disposed."""
    first = start(4)
    with pytest.raises(BusyTriggerError, match="already has a live LK session"):
        native.NativeSession.start(native.NativeConfig(num_workers=4))
    first.dispose()
    second = start(4)
    second.dispose()


@pytest.mark.parametrize("kw", [dict(poll_replicas=2), dict(poll_replicas=4, poll_mode="gateway")])
def test_removed_replica_knobs_are_refused(kw):
    """Replicated to_gpu cells / event rings were measured slower and removed
    (DESIGN.md section 3): lk_create refuses them instead of ignoring them."""
    from paper_2310_01212_b200.errors import ConfigError
    with pytest.raises(ConfigError, match="poll_replicas must be 1"):
        native.NativeSession.start(native.NativeConfig(num_workers=4, **kw))
    start(4).dispose()   # and the device is free for the next session


@pytest.mark.slow
def test_gateway_event_tags_wrap():
    """More than 2^16 ring events (the torn-read tag is seq & 0xFFFF) and
    hundreds of ring wraparounds: every round still completes in order."""
    session = start(16, poll_mode="gateway")
    session.register(WorkDescriptor(slot=0, kind="empty"))
    full = (1 << 16) - 1
    _, done, cyc = session.bench_roundtrip([full], 0, 36_000)   # 2 events per round
    assert (cyc >= done).all() and len(done) == 36_000
    session.dispose()


def test_sm_topology_groups_sms_by_gpc():
    """lk_sm_topology: clustered probe launches group every SM into GPCs
    (B200: 148 SMs in ~8 GPCs of <= 20); a session's workers map onto them."""
    topo = native.sm_topology(0)
    assert len(topo) >= 148 and all(g >= 0 for g in topo)
    sizes = {}
    for g in topo:
        sizes[g] = sizes.get(g, 0) + 1
    assert 2 <= len(sizes) <= 32 and max(sizes.values()) <= 32, sizes
    session = start(None)
    by = native.workers_by_gpc(session.smid_map, topo)
    session.dispose()
    assert sum(len(v) for v in by.values()) == session.num_workers and -1 not in by


def test_huge_slot_numbers_are_refused_cleanly():
    """Slots up to the reference's MAX_SLOT (2^32 - 17) are legal words; ones
    beyond the device table are a UsageError, not a ctypes overflow."""
    session = start(1)
    with pytest.raises(UsageError):
        session.trigger(1, WorkDescriptor(slot=protocol.MAX_SLOT, iterations=1))
    session.trigger(1, TINY_WORK)
    session.wait(1)
    session.dispose()


def test_profile_run_completes_and_frees_the_device():
    """lk_profile_run: a session driven by the internal host thread boots,
    runs its handshakes, exits and releases the device claim (a normal
    session starts right after)."""
    ns = native.profile_run(native.NativeConfig(num_workers=16), 2000)
    assert ns > 0
    s = start(4)
    s.trigger(1, TINY_WORK)
    s.wait(1)
    s.dispose()
    assert_trace_ok(s)


def test_profile_run_payload_dispatches():
    """lk_profile_run with payload descriptors: full-mask dispatches of each
    in turn; three in-place saxpy passes equal the oracle applied three times."""
    from oracle import work as W
    from paper_2310_01212_b200.device import DeviceBuffer
    n = 100_003
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y = rng.uniform(-1, 1, n).astype(np.float32)
    dx, dy = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y)
    try:
        w = WorkDescriptor(slot=1, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=dy, alpha=0.5)
        assert native.profile_run(native.NativeConfig(num_workers=32), 3, [w]) > 0
        want = y
        for _ in range(3):
            want = W.saxpy_f32(0.5, x, want)
        np.testing.assert_array_equal(dy.download(np.float32, n).view(np.uint32), want.view(np.uint32))
    finally:
        dx.free()
        dy.free()


def test_adaptive_ack_delay_lands_the_ack_on_the_first_load():
    """DIRECT, default ack delay: after a warm-up the worker's first load
    after FINISHED sees the host's NOP (timeline word 10 = loads issued while
    awaiting the ack); with the delay off the first load always misses."""
    def ack_loads(**kw):
        s, _ = native.NativeSession.start(native.NativeConfig(num_workers=16, spin_strategy=native.PURE_SPIN,
                                                              timeline=True, **kw))
        try:
            s.register(WorkDescriptor(slot=0, kind="empty"))
            s.bench_roundtrip([1 << i for i in range(16)], 0, 16 * 400)
            return s.last_timeline()[:, 10].astype(int)
        finally:
            s.close()
    with_delay = ack_loads()
    without = ack_loads(ack_delay_ns=0)
    assert np.median(with_delay) == 1, with_delay
    assert np.median(without) >= 2, without


def test_abort_after_worker_death_reclaims_the_device():
    """A dead worker leaves the session unusable; abort() retires the kernel
    (EXIT to the survivors), close() frees it, and the device takes a new
    session at once (the one-session claim is released)."""
    session = start(4)
    _lib.check(session._lib.lk_debug_poke(session._h, 2, 9))
    session._spin_until(lambda: session.worker_phase[2] is protocol.Phase.EXITED, "device exit", [2])
    with pytest.raises(UsageError, match="worker 2 died"):
        session.trigger(0b0001, TINY_WORK)
    session.abort(timeout_s=5.0)
    assert not session._kernel_alive()
    session.close()
    _LIVE.remove(session)
    fresh = start(4)
    fresh.trigger(0b1111, TINY_WORK)
    fresh.wait(0b1111)
    fresh.dispose()
    assert_trace_ok(fresh)


def test_wait_timeout_raises_hang_then_a_later_wait_completes():
    """lk_wait's C-side spin honours wait_timeout (native.py:233-248): work
    that outlasts it raises HangDetected naming the workers, the dispatch
    stays pending, and a later wait collects it once the worker finishes."""
    session = start(1, wait_timeout_s=0.02)
    session.trigger(1, WorkDescriptor(slot=0, iterations=60_000_000))
    with pytest.raises(HangDetected) as ei:
        session.wait(1)
    assert ei.value.sm_ids == (0,)
    assert session.pending_mask == 1
    for _ in range(500):
        try:
            session.wait(1)
            break
        except HangDetected:
            continue
    else:
        pytest.fail("the long task never finished")
    assert session.pending_mask == 0
    session.dispose()
    assert_trace_ok(session)


def test_cached_descriptor_fast_path_runs_the_work():
    """LK_HINT_CACHED: re-dispatching the same staged busy_loop descriptor to
    the same worker skips the descriptor fetch and runs the loop on the fast
    path -- the iterations still all execute, a restaged slot is fetched
    again, and the handshakes stay legal."""
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=2, spin_strategy=native.PURE_SPIN))
    _LIVE.append(s)
    cyc = {}
    for n in (100_000, 1_000_000):
        w = WorkDescriptor(slot=3, iterations=n)
        for rep in range(3):                      # rep 0 fetches, reps 1-2 reuse the cache
            s.trigger(1, w)
            s.wait(1)
            t = s.last_timeline().astype(np.int64)
            cyc[(n, rep)] = int(t[0, 7] - t[0, 6])
    for n in (100_000, 1_000_000):
        for rep in range(3):
            assert cyc[(n, rep)] >= n, cyc
    assert cyc[(1_000_000, 2)] > 5 * cyc[(100_000, 2)], cyc
    assert cyc[(1_000_000, 0)] > 5 * cyc[(100_000, 2)], cyc   # restaged slot 3: no stale copy
    # payload kinds through the cache: same descriptor and mask twice, both exact
    from oracle import work as W
    from paper_2310_01212_b200.device import DeviceBuffer
    a = np.arange(4096, dtype=np.int32)
    da, db, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(a), DeviceBuffer(4 * 4096)
    try:
        w = WorkDescriptor(slot=5, kind="vector_add_i32", data_in_ref=(da, db), data_out_ref=do)
        for rep in range(2):
            do.upload(np.zeros(4096, dtype=np.int32))
            s.trigger(0b11, w)
            s.wait(0b11)
            np.testing.assert_array_equal(do.download(np.int32, 4096), W.vector_add_i32(a, a))
    finally:
        for b in (da, db, do):
            b.free()
    s.dispose()
