"""Sessions with the descriptor table in pinned mapped host memory
(NativeConfig.host_descriptors / LK_CF_HOST_DESC): register, trigger and wait
make no CUDA call, which is what keeps a session usable under a profiler that
serialises launches.  Same results and traces as the device-table sessions."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import projection
from oracle import protocol as O
from oracle import work as W
from paper_2310_01212_b200 import host, native
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor
from paper_2310_01212_b200.errors import ConfigError

pytestmark = pytest.mark.gpu


def test_host_descriptors_need_direct_mode():
    with pytest.raises(ConfigError):
        native.NativeSession.start(native.NativeConfig(num_workers=4, host_descriptors=True, poll_mode="gateway"))


def test_host_descriptor_payloads_and_restage():
    nw = 48
    n = 300_001
    a = np.random.default_rng(0).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    b = np.random.default_rng(1).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    x = np.random.default_rng(2).uniform(-1, 1, n).astype(np.float32)
    y = np.random.default_rng(3).uniform(-1, 1, n).astype(np.float32)
    da, db, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(b), DeviceBuffer(4 * n)
    dx, dy, dz = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y), DeviceBuffer(4 * n)
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=nw, host_descriptors=True,
                                                          record_trace=True, trace_capacity=2048))
    program = []
    try:
        full = host.full_mask(nw)
        half = host.mask_of(range(0, nw, 2))
        s.trigger(full, WorkDescriptor(slot=4, kind="vector_add_i32", data_in_ref=(da, db), data_out_ref=do))
        s.wait(full)
        program.append((full, 4))
        np.testing.assert_array_equal(do.download(np.int32, n), W.vector_add_i32(a, b))
        # the same slot re-staged with another kind and another mask: the
        # workers must see the new host-side descriptor, not a stale copy
        s.trigger(half, WorkDescriptor(slot=4, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=dz, alpha=-0.25))
        s.wait(half)
        program.append((half, 4))
        np.testing.assert_array_equal(dz.download(np.float32, n).view(np.uint32),
                                      W.saxpy_f32(-0.25, x, y).view(np.uint32))
        for k in range(3 * nw):
            m = 1 << (k % nw)
            s.trigger(m, WorkDescriptor(slot=0, kind="empty"))
            s.wait(m)
            program.append((m, 0))
        s.dispose()
        writes = [(r.side, r.sm_id, r.word) for r in s.recorded_trace()]
        assert O.replay(writes).violation is None
        per = projection.program_slots(program, nw)
        proj = projection.projections(writes, nw)
        for i in range(nw):
            assert proj[i] == projection.expected_projection(per[i]), i
    finally:
        s.close()
        for buf in (da, db, do, dx, dy, dz):
            buf.free()
