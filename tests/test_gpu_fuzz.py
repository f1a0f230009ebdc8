"""Seeded randomized programs against the B200 session: random poll modes and
payload paths, overlapping dispatches on disjoint worker sets, partial waits,
every payload kind at random sizes and masks, about a third of the buffers in
host-mapped memory (zero-copy).  Each result is checked against
the oracle and each session's full trace is replayed by the oracle validator
and checked against the golden per-worker projection."""
from __future__ import annotations

import random

import numpy as np
import pytest

from oracle import projection
from oracle import protocol as O
from oracle import work as W
from paper_2310_01212_b200 import host, native
from paper_2310_01212_b200.device import DeviceBuffer, HostBuffer, WorkDescriptor, reduce_blocks

pytestmark = pytest.mark.gpu

NW = 24


def _check_trace(session, program):
    writes = [(r.side, r.sm_id, r.word) for r in session.recorded_trace()]
    r = O.replay(writes)
    assert r.violation is None, r.violation
    per = projection.program_slots(program, NW)
    proj = projection.projections(writes, NW)
    for i in range(NW):
        assert proj[i] == projection.expected_projection(per[i]), i


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6, 7, 8])
def test_random_programs(seed):
    rng = random.Random(seed)
    cfg = native.NativeConfig(num_workers=NW, record_trace=True, trace_capacity=8192,
                              poll_mode=rng.choice(["direct", "gateway", "hybrid"]),
                              tma_payload=rng.random() < 0.8, lazy_ack=rng.random() < 0.3,
                              ring_stages=rng.choice([2, 4, 6]),
                              tma_min_workers=rng.choice([1, 4, 49]))
    s, _ = native.NativeSession.start(cfg)
    nrng = np.random.default_rng(seed)
    bufs = []
    try:
        program = []
        slot = 0
        for step in range(60):
            # up to three overlapping dispatches on disjoint worker sets, then wait
            free = list(range(NW))
            rng.shuffle(free)
            active = []
            for _ in range(rng.randint(1, 3)):
                if not free:
                    break
                k = rng.randint(1, min(len(free), 8))
                ids, free = free[:k], free[k:]
                mask = host.mask_of(ids)
                kind = rng.choice(["empty", "busy", "vector_add_i32", "saxpy_f32", "block_reduce_f32",
                                   "hbm_stream"])
                n = rng.choice([1, 5, 32, 1000, 65536 + rng.randrange(100), 300_001])
                check = None
                # about a third of the payload buffers are zero-copy host-mapped memory
                host_side = rng.random() < 0.35

                def mk(arr=None, nbytes=0, host_ok=True):
                    cls = HostBuffer if (host_side and host_ok) else DeviceBuffer
                    return cls.from_array(arr) if arr is not None else cls(nbytes)
                if kind == "empty":
                    w = WorkDescriptor(slot=slot, kind="empty")
                elif kind == "busy":
                    w = WorkDescriptor(slot=slot, iterations=rng.randrange(2000))
                elif kind == "vector_add_i32":
                    a = nrng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
                    b = nrng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
                    da, db, do = mk(a), DeviceBuffer.from_array(b), mk(nbytes=4 * n)
                    bufs += [da, db, do]
                    w = WorkDescriptor(slot=slot, kind=kind, data_in_ref=(da, db), data_out_ref=do)
                    check = lambda do=do, a=a, b=b, n=n: np.testing.assert_array_equal(  # noqa: E731
                        do.download(np.int32, n), W.vector_add_i32(a, b))
                elif kind == "saxpy_f32":
                    x = nrng.uniform(-1, 1, n).astype(np.float32)
                    y = nrng.uniform(-1, 1, n).astype(np.float32)
                    dx, dy = mk(x), mk(y)
                    bufs += [dx, dy]
                    alpha = float(rng.choice([1.5, -0.25, 3.0]))
                    w = WorkDescriptor(slot=slot, kind=kind, data_in_ref=(dx, dy), data_out_ref=dy, alpha=alpha)
                    check = lambda dy=dy, x=x, y=y, n=n, alpha=alpha: np.testing.assert_array_equal(  # noqa: E731
                        dy.download(np.float32, n).view(np.uint32), W.saxpy_f32(alpha, x, y).view(np.uint32))
                elif kind == "block_reduce_f32":
                    x = nrng.integers(0, 8, n).astype(np.float32)
                    nbk = reduce_blocks(n)
                    dx, dp, dt = mk(x), DeviceBuffer(8 * nbk), mk(nbytes=8)   # partials: device memory
                    bufs += [dx, dp, dt]
                    w = WorkDescriptor(slot=slot, kind=kind, data_in_ref=dx, data_out_ref=dp, total_ref=dt)

                    def check(dp=dp, dt=dt, x=x, nbk=nbk):
                        np.testing.assert_array_equal(dp.download(np.float64, nbk), W.block_reduce_partials(x))
                        assert dt.download(np.float64, 1)[0] == W.block_reduce_total(x)
                else:
                    src = nrng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
                    ds, dd = mk(src), mk(nbytes=4 * n, host_ok=rng.random() < 0.5)
                    bufs += [ds, dd]
                    w = WorkDescriptor(slot=slot, kind=kind, data_in_ref=ds, data_out_ref=dd,
                                       iterations=rng.randint(1, 2))
                    check = lambda dd=dd, src=src, n=n: np.testing.assert_array_equal(  # noqa: E731
                        dd.download(np.int32, n), src)
                s.trigger(mask, w)
                program.append((mask, slot))
                active.append((mask, check))
                slot += 1
            rng.shuffle(active)
            for mask, check in active:
                s.wait(mask)
                if check is not None:
                    check()
        s.dispose()
        _check_trace(s, program)
    finally:
        s.close()
        for b in bufs:
            b.free()
