"""Several host threads driving one session (the multi-driver throughput
setup).  Own module: a live session owns every SM, so this must not overlap
another module's session fixture."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import work as W
from paper_2310_01212_b200 import host, native
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor

pytestmark = pytest.mark.gpu


def _i32(n, seed):
    return np.random.default_rng(seed).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)


@pytest.mark.parametrize("mode", ["direct", "hybrid"])
def test_concurrent_host_threads_on_disjoint_workers(mode):
    """Four host threads drive disjoint worker groups of one session at once
    (the multi-driver throughput setup), each dispatching payloads on its own
    slots and checking every result against the oracle; the merged trace
    still validates."""
    import threading
    from oracle import protocol as O
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, poll_mode=mode, record_trace=True,
                                                          trace_capacity=4096))
    try:
        n = s.num_workers
        groups = [list(range(g, n, 4)) for g in range(4)]
        errors = []

        def drive(g):
            try:
                rng = np.random.default_rng(100 + g)
                el = 50_000 + g
                a, b = _i32(el, 10 + g), _i32(el, 20 + g)
                da, db, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(b), DeviceBuffer(4 * el)
                want = W.vector_add_i32(a, b)
                for k in range(25):
                    ids = groups[g] if k % 2 == 0 else [int(rng.choice(groups[g]))]
                    m = host.mask_of(ids)
                    if k % 3 == 0:
                        w = WorkDescriptor(slot=100 * (g + 1) + k, kind="empty")
                    else:
                        w = WorkDescriptor(slot=100 * (g + 1) + k, kind="vector_add_i32", data_in_ref=(da, db),
                                           data_out_ref=do)
                    s.trigger(m, w)
                    s.wait(m)
                    if w.kind == "vector_add_i32":
                        np.testing.assert_array_equal(do.download(np.int32, el), want)
                        do.upload(np.zeros(el, np.int32))
            except Exception as exc:   # surfaced below
                errors.append(exc)

        ths = [threading.Thread(target=drive, args=(g,)) for g in range(4)]
        for t in ths:
            t.start()
        for t in ths:
            t.join(timeout=120)
        assert not errors, errors
        s.dispose()
        r = O.replay([(x.side, x.sm_id, x.word) for x in s.recorded_trace()])
        assert r.violation is None, r.violation
    finally:
        s.close()
