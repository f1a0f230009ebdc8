"""The TMA ring's positions (kept modulo 2 x stages, lk_kernels.cu rp_*)
across many dispatches: for several ring depths, and with the producer and
the consumers in one warp (threads_per_worker=32), a long run of saxpy,
hbm_stream and block_reduce dispatches whose per-worker tile counts vary
from 1 to ~40, so that every dispatch starts the two rings (the maps' shared
ring and the reduce's owner-warp ring) at a different stage and phase.
Every result is checked against the oracle bit for bit."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import work as W
from paper_2310_01212_b200 import host, native
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor, reduce_blocks

pytestmark = pytest.mark.gpu

NW = 8


@pytest.mark.parametrize("stages,threads", [(2, 512), (3, 512), (5, 512), (7, 512), (12, 512), (5, 32)])
def test_ring_positions_many_dispatches(stages, threads):
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=NW, ring_stages=stages,
                                                          threads_per_worker=threads, tma_min_workers=1))
    rng = np.random.default_rng(stages * 100 + threads)
    full = host.full_mask(NW)
    nmax = NW * 40 * 4096 + 77
    bufs = []
    try:
        dx, dy = DeviceBuffer(4 * nmax), DeviceBuffer(4 * nmax)
        dp, dt = DeviceBuffer(8 * reduce_blocks(nmax)), DeviceBuffer(8)
        bufs += [dx, dy, dp, dt]
        sizes = [int(rng.integers(1, nmax)) for _ in range(36)] + [4096 * NW, 4096 * NW + 1, 17, nmax]
        for k, n in enumerate(sizes):
            x = rng.uniform(-1, 1, n).astype(np.float32)
            y = rng.uniform(-1, 1, n).astype(np.float32)
            dx.upload(x)
            dy.upload(y)
            kind = ("saxpy_f32", "hbm_stream", "block_reduce_f32")[k % 3]
            if kind == "saxpy_f32":
                w = WorkDescriptor(slot=1, kind=kind, data_in_ref=(dx, dy), data_out_ref=dy, alpha=0.5, n=n)
            elif kind == "hbm_stream":
                w = WorkDescriptor(slot=2, kind=kind, iterations=1 + k % 2, data_in_ref=dx, data_out_ref=dy, n=n)
            else:
                w = WorkDescriptor(slot=3, kind=kind, data_in_ref=dx, data_out_ref=dp, total_ref=dt, n=n)
            s.trigger(full, w)
            s.wait(full)
            if kind == "saxpy_f32":
                np.testing.assert_array_equal(dy.download(np.float32, n).view(np.uint32),
                                              W.saxpy_f32(0.5, x, y).view(np.uint32), err_msg=f"dispatch {k}, n={n}")
            elif kind == "hbm_stream":
                np.testing.assert_array_equal(dy.download(np.float32, n).view(np.uint32),
                                              W.hbm_stream(x).view(np.uint32), err_msg=f"dispatch {k}, n={n}")
            else:
                np.testing.assert_array_equal(dp.download(np.float64, reduce_blocks(n)), W.block_reduce_partials(x),
                                              err_msg=f"dispatch {k}, n={n}")
                assert dt.download(np.float64, 1)[0] == W.block_reduce_total(x), (k, n)
        s.dispose()
    finally:
        s.close()
        for b in bufs:
            b.free()
