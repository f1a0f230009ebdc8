"""The conventional launch+sync baseline (ThreadSpawnBaseline analogue,
native.py:304-331) runs the same device work functions; it must produce the
oracle's results through both payload paths (TMA bulk ring and LSU loads).

Kept in its own module: an LK session owns every SM (one resident CTA each,
registers and shared memory sized for exactly one), so a baseline kernel can
only be scheduled when no session is live."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import work as W
from paper_2310_01212_b200 import native
from paper_2310_01212_b200.device import DeviceBuffer, HostBuffer, WorkDescriptor, reduce_blocks

pytestmark = pytest.mark.gpu


def _i32(n, seed):
    return np.random.default_rng(seed).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)


def _f32(n, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, n).astype(np.float32)


@pytest.mark.parametrize("tma", [True, False])
@pytest.mark.parametrize("n", [65536, 1000003, 37])
def test_baseline_kernel_same_results(tma, n):
    b = native.LaunchSyncBaseline(tma_payload=tma)
    a, c = _i32(n, 0), _i32(n, 1)
    da, dc, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(c), DeviceBuffer(4 * n)
    b.launch(WorkDescriptor(slot=0, kind="vector_add_i32", data_in_ref=(da, dc), data_out_ref=do))
    b.wait()
    np.testing.assert_array_equal(do.download(np.int32, n), W.vector_add_i32(a, c))
    x, y = _f32(n, 2), _f32(n, 3)
    dx, dy, dz = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y), DeviceBuffer(4 * n)
    b.launch(WorkDescriptor(slot=0, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=dz, alpha=1.5))
    b.wait()
    np.testing.assert_array_equal(dz.download(np.float32, n).view(np.uint32),
                                  W.saxpy_f32(1.5, x, y).view(np.uint32))
    xi = np.random.default_rng(9).integers(0, 8, n).astype(np.float32)
    dxi, dp, dt = DeviceBuffer.from_array(xi), DeviceBuffer(8 * max(1, reduce_blocks(n))), DeviceBuffer(8)
    b.launch(WorkDescriptor(slot=0, kind="block_reduce_f32", data_in_ref=dxi, data_out_ref=dp, total_ref=dt))
    b.wait()
    np.testing.assert_array_equal(dp.download(np.float64, reduce_blocks(n)), W.block_reduce_partials(xi))
    assert dt.download(np.float64, 1)[0] == W.block_reduce_total(xi)
    xu = _f32(n, 21)
    dxu = DeviceBuffer.from_array(xu)
    b.launch(WorkDescriptor(slot=0, kind="block_reduce_f32", data_in_ref=dxu, data_out_ref=dp, total_ref=dt))
    b.wait()   # the same bits as the persistent kernel's reduce: one definition
    assert dt.download(np.float64, 1)[0] == W.block_reduce_total(xu)
    b.close()


def test_baseline_time_kernel_reports_positive():
    n = 1 << 20
    b = native.LaunchSyncBaseline()
    x, y = DeviceBuffer(4 * n), DeviceBuffer(4 * n)
    ms = b.time_kernel(WorkDescriptor(slot=0, kind="saxpy_f32", data_in_ref=(x, y), data_out_ref=y), 3)
    assert 0 < ms < 100
    b.close()


def test_baseline_runs_beside_a_partitioned_session():
    """An sm_partition session leaves the other SMs to ordinary kernels: the
    baseline launches (and synchronizes) while the persistent kernel is
    resident, both produce the oracle's results, and the session keeps
    answering in between."""
    session, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, sm_partition=16, record_trace=True))
    try:
        b = native.LaunchSyncBaseline(beside=session)
        assert b.grid == session.partition_info[1]
        n = 1 << 20
        a, c = _i32(n, 0), _i32(n, 1)
        da, dc, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(c), DeviceBuffer(4 * n)
        for k in range(5):
            b.launch(WorkDescriptor(slot=0, kind="vector_add_i32", data_in_ref=(da, dc), data_out_ref=do))
            session.trigger(1 << (k % session.num_workers), WorkDescriptor(slot=0, kind="empty"))
            session.wait(1 << (k % session.num_workers))
            b.wait()
        np.testing.assert_array_equal(do.download(np.int32, n), W.vector_add_i32(a, c))
        x, y = _f32(n, 2), _f32(n, 3)
        dx, dy = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y)
        ms = b.time_kernel(WorkDescriptor(slot=0, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=dy,
                                          alpha=1.5), 1)
        assert ms > 0
        np.testing.assert_array_equal(dy.download(np.float32, n).view(np.uint32),
                                      W.saxpy_f32(1.5, x, y).view(np.uint32))
        b.close()
        session.dispose()
        from oracle import protocol as O
        assert O.replay([(r.side, r.sm_id, r.word) for r in session.recorded_trace()]).violation is None
    finally:
        session.close()


@pytest.mark.parametrize("mode", ["kernel_sync", "kernel_query", "graph_sync"])
def test_launch_floor_modes_run(mode):
    """The cheapest conventional launch+sync flows (the ≥5x denominator's
    candidates) each complete every task: completion is observed after the
    launch call returns, and no task takes a whole second."""
    total, launch = native.launch_floor(0, mode, 500)
    assert (total >= launch).all()
    assert int(total.max()) < 1_000_000_000
    assert np.median(total) > 0


def test_launch_floor_spin_schedule():
    total, _ = native.launch_floor(0, "kernel_sync", 200, spin_sched=True)
    assert np.median(total) > 0


def test_launch_sync_baseline_with_host_buffers():
    """Zero-copy buffers through the conventional launch (LK_DF_HOSTMEM
    classified at launch, like a staged descriptor)."""
    n = 4100
    a, b = _i32(n, 7), _i32(n, 8)
    ha, hb, ho = HostBuffer.from_array(a), HostBuffer.from_array(b), HostBuffer(4 * n)
    base = native.LaunchSyncBaseline()
    try:
        base.launch(WorkDescriptor(slot=0, kind="vector_add_i32", data_in_ref=(ha, hb), data_out_ref=ho))
        base.wait()
    finally:
        base.close()
    np.testing.assert_array_equal(ho.array(np.int32, n), W.vector_add_i32(a, b))
