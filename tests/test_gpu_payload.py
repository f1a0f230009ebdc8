"""Payload work items on the persistent workers vs the numpy oracle.

Bars: integer work bit-exact; SAXPY bit-exact (the
device uses __fmul_rn/__fadd_rn, numpy computes fl(fl(a*x)+y)); reduction
exact on small-integer data and rtol 1e-6 against a float64 sum on U[0,1).
Inputs are seeded (default_rng(0/1) for int32, (2/3) for fp32, alpha=1.5).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import work as W
from paper_2310_01212_b200 import host, native
from paper_2310_01212_b200.device import DeviceBuffer, WorkDescriptor, reduce_blocks
from paper_2310_01212_b200.errors import ConfigError

pytestmark = pytest.mark.gpu

RTOL_F32_REDUCE = 1e-6


# "tma": the ring for dispatches to >= 49 workers, LSU loads below (the
# default); "ring": the ring for every dispatch (tma_min_workers=1)
@pytest.fixture(scope="module", params=["tma-direct", "ring-direct", "lsu-direct", "tma-gateway", "ring-hybrid"])
def session(request):
    try:   # bring torch's CUDA state AND the kernels the torch test uses up before the
        # persistent kernel is resident: CUDA 12 loads kernels lazily, and a module
        # load while a spinning kernel is resident waits on it forever.
        import torch
        t = torch.arange(8, dtype=torch.int32, device="cuda")
        (t + 1).float().cpu()
        torch.empty_like(t).copy_(t)
        torch.cuda.synchronize()
    except Exception:
        pass
    path, mode = request.param.split("-")
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_yield_threshold=200, poll_mode=mode,
                                                          tma_payload=path != "lsu",
                                                          tma_min_workers=1 if path == "ring" else 49))
    yield s
    s.close()


def _i32(n, seed):
    return np.random.default_rng(seed).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)


def _f32(n, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, n).astype(np.float32)


def run(session, mask, work):
    session.trigger(mask, work)
    session.wait(mask)


MASKS = {"one": lambda n: 1, "four": lambda n: 0b1111, "odd": lambda n: sum(1 << i for i in range(1, n, 3)),
         "full": lambda n: host.full_mask(n)}


@pytest.mark.parametrize("mask_name", list(MASKS))
@pytest.mark.parametrize("n", [65536, 1, 31, 33, 1000003])
def test_vector_add_i32_bit_exact(session, mask_name, n):
    a, b = _i32(n, 0), _i32(n, 1)
    da, db, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(b), DeviceBuffer(4 * n)
    run(session, MASKS[mask_name](session.num_workers),
        WorkDescriptor(slot=10, kind="vector_add_i32", data_in_ref=(da, db), data_out_ref=do, n=n))
    np.testing.assert_array_equal(do.download(np.int32, n), W.vector_add_i32(a, b))


def test_vector_add_wraparound_edges(session):
    a = np.array([2**31 - 1, -2**31, -1, 0, 2**31 - 1] * 7, dtype=np.int32)
    b = np.array([1, -1, 1, 0, 2**31 - 1] * 7, dtype=np.int32)
    da, db, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(b), DeviceBuffer(a.nbytes)
    run(session, 0b11, WorkDescriptor(slot=11, kind="vector_add_i32", data_in_ref=(da, db), data_out_ref=do,
                                       n=len(a)))
    np.testing.assert_array_equal(do.download(np.int32, len(a)), W.vector_add_i32(a, b))


def test_misaligned_pointers_take_scalar_path(session):
    n = 1001
    a, b = _i32(n + 1, 4), _i32(n + 1, 5)
    da, db, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(b), DeviceBuffer(4 * (n + 1))
    work = WorkDescriptor(slot=12, kind="vector_add_i32", data_in_ref=(da.ptr + 4, db.ptr + 4),
                          data_out_ref=do.ptr + 4, n=n)
    assert work.to_c().flags & 1
    run(session, 0b111, work)
    np.testing.assert_array_equal(do.download(np.int32, n + 1)[1:], W.vector_add_i32(a[1:], b[1:]))


@pytest.mark.parametrize("n", [1, 33, 1 << 18, 12345, 4 << 20])
def test_saxpy_f32_bit_exact_in_place(session, n):
    x, y = _f32(n, 2), _f32(n, 3)
    dx, dy = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y)
    mask = host.full_mask(session.num_workers)
    run(session, mask, WorkDescriptor(slot=20, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=dy,
                                      alpha=1.5))
    want = W.saxpy_f32(1.5, x, y)
    np.testing.assert_array_equal(dy.download(np.float32, n).view(np.uint32), want.view(np.uint32))
    # a second dispatch re-reads what the first wrote (L1/L2 coherence across dispatches)
    run(session, mask, WorkDescriptor(slot=21, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=dy,
                                      alpha=1.5))
    want2 = W.saxpy_f32(1.5, x, want)
    np.testing.assert_array_equal(dy.download(np.float32, n).view(np.uint32), want2.view(np.uint32))


@pytest.mark.parametrize("kind", ["vector_add_i32", "saxpy_f32", "hbm_stream"])
@pytest.mark.parametrize("mask_name", ["one", "odd", "full"])
@pytest.mark.parametrize("n", [31, 4097, 300_007])
def test_map_writes_stop_at_n(session, kind, mask_name, n):
    """The last worker's shard ends at n: the output's guard words past n
    (inside the same allocation) are never written, whatever the shard
    boundaries and the path (ring tiles, LSU tails)."""
    pad = 64
    guard = np.int32(0x5A5A5A5A)
    if kind == "saxpy_f32":   # finite floats: NaN payloads differ between numpy and the device
        a, b = _f32(n + pad, 7).view(np.int32), _f32(n + pad, 8).view(np.int32)
    else:
        a, b = _i32(n + pad, 7), _i32(n + pad, 8)
    out = np.full(n + pad, guard, np.int32)
    da, db, do = DeviceBuffer.from_array(a), DeviceBuffer.from_array(b), DeviceBuffer.from_array(out)
    ins = da if kind == "hbm_stream" else (da, db)
    run(session, MASKS[mask_name](session.num_workers),
        WorkDescriptor(slot=48, kind=kind, data_in_ref=ins, data_out_ref=do, n=n, alpha=1.5))
    got = do.download(np.int32, n + pad)
    np.testing.assert_array_equal(got[n:], out[n:])
    if kind == "vector_add_i32":
        want = W.vector_add_i32(a[:n], b[:n])
    elif kind == "saxpy_f32":
        want = W.saxpy_f32(1.5, a[:n].view(np.float32), b[:n].view(np.float32)).view(np.int32)
    else:
        want = a[:n]
    np.testing.assert_array_equal(got[:n], want)


def test_saxpy_after_host_rewrite_is_coherent(session):
    """Copyin between dispatches (DMA into L2) must be seen by the workers."""
    n = 1 << 16
    x, y = _f32(n, 6), _f32(n, 7)
    dx, dy, do = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y), DeviceBuffer(4 * n)
    work = WorkDescriptor(slot=22, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=do, alpha=-0.75)
    run(session, 0b1, work)
    x2 = _f32(n, 8)
    session.copyin(dx, x2)
    run(session, 0b1, work)
    np.testing.assert_array_equal(do.download(np.float32, n), W.saxpy_f32(-0.75, x2, y))


def _reduce(session, mask, x, slot):
    n = x.size
    dx, dp, dt = DeviceBuffer.from_array(x), DeviceBuffer(8 * max(1, reduce_blocks(n))), DeviceBuffer(8)
    run(session, mask, WorkDescriptor(slot=slot, kind="block_reduce_f32", data_in_ref=dx, data_out_ref=dp,
                                      total_ref=dt))
    parts = dp.download(np.float64, reduce_blocks(n))
    tot = dt.download(np.float64, 1)[0]
    for b in (dx, dp, dt):
        b.free()
    return parts, tot


@pytest.mark.parametrize("workers", [1, 7, 148])
def test_block_reduce_exact_on_small_integers(session, workers):
    n = 3_000_017
    x = np.random.default_rng(9).integers(0, 8, n).astype(np.float32)
    parts, tot = _reduce(session, host.full_mask(workers), x, 30)
    np.testing.assert_array_equal(parts, W.block_reduce_partials(x))
    assert tot == W.block_reduce_total(x) == float(x.astype(np.float64).sum())


@pytest.mark.parametrize("n", [0, 1, 3, 4095, 4096, 4097, 4099, 8192 + 2, 1_048_573, 9_000_003])
def test_block_reduce_bit_exact_any_size(session, n):
    """Block partials and total bit-identical to the oracle's fixed order of
    operations on U[-1,1) data, for sizes around the block and vector edges
    (tail-only last blocks included)."""
    x = _f32(n, 11)
    parts, tot = _reduce(session, host.full_mask(session.num_workers), x, 32)
    np.testing.assert_array_equal(parts.view(np.uint64), W.block_reduce_partials(x).view(np.uint64))
    assert np.float64(tot).view(np.uint64) == np.float64(W.block_reduce_total(x)).view(np.uint64)


def test_block_reduce_uniform_within_rtol(session):
    n = 16 << 20   # 64 MiB of fp32
    x = _f32(n, 10, 0.0, 1.0)
    mask = host.full_mask(session.num_workers)
    parts, tot = _reduce(session, mask, x, 31)
    np.testing.assert_array_equal(parts, W.block_reduce_partials(x))
    np.testing.assert_allclose(tot, float(x.astype(np.float64).sum()), rtol=RTOL_F32_REDUCE)
    assert tot == W.block_reduce_total(x)
    # the result does not depend on the worker set or the schedule: any mask,
    # any run, the same bits (dynamic block claiming)
    for m in (mask, host.mask_of(range(0, session.num_workers, 3)), 0b1011):
        p2, t2 = _reduce(session, m, x, 31)
        assert t2 == tot
        np.testing.assert_array_equal(p2, parts)


def test_block_reduce_misaligned_input(session):
    n = 100_003
    base = _f32(n + 1, 13)
    dbase = DeviceBuffer.from_array(base)
    dp, dt = DeviceBuffer(8 * reduce_blocks(n)), DeviceBuffer(8)
    run(session, host.full_mask(session.num_workers),
        WorkDescriptor(slot=33, kind="block_reduce_f32", data_in_ref=dbase.ptr + 4, n=n, data_out_ref=dp,
                       total_ref=dt))
    np.testing.assert_array_equal(dp.download(np.float64, reduce_blocks(n)), W.block_reduce_partials(base[1:]))
    assert dt.download(np.float64, 1)[0] == W.block_reduce_total(base[1:])


def test_block_reduce_short_partials_buffer_refused(session):
    x = DeviceBuffer(4 * 10_000)
    with pytest.raises(ConfigError):
        WorkDescriptor(slot=34, kind="block_reduce_f32", data_in_ref=x, data_out_ref=DeviceBuffer(8),
                       total_ref=DeviceBuffer(8)).to_c()


@pytest.mark.parametrize("passes", [1, 3])
def test_hbm_stream_copies(session, passes):
    n = (1 << 20) + 7
    src = _i32(n, 12)
    ds, dd = DeviceBuffer.from_array(src), DeviceBuffer(4 * n)
    run(session, host.full_mask(session.num_workers),
        WorkDescriptor(slot=40, kind="hbm_stream", iterations=passes, data_in_ref=ds, data_out_ref=dd))
    np.testing.assert_array_equal(dd.download(np.int32, n), src)


def test_full_size_saxpy_64mib_matches_oracle(session):
    """BASELINE config 3 at its largest size (64 MiB per vector), bit-exact."""
    n = 16 << 20
    x, y = _f32(n, 2), _f32(n, 3)
    dx, dy, do = DeviceBuffer.from_array(x), DeviceBuffer.from_array(y), DeviceBuffer(4 * n)
    run(session, host.full_mask(session.num_workers),
        WorkDescriptor(slot=50, kind="saxpy_f32", data_in_ref=(dx, dy), data_out_ref=do, alpha=1.5))
    np.testing.assert_array_equal(do.download(np.float32, n).view(np.uint32),
                                  W.saxpy_f32(1.5, x, y).view(np.uint32))


def test_torch_tensors_as_payload_refs(session):
    torch = pytest.importorskip("torch")
    n = 100_000
    a, b = _i32(n, 0), _i32(n, 1)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    to = torch.empty_like(ta)
    torch.cuda.current_stream().synchronize()
    run(session, 0b11, WorkDescriptor(slot=60, kind="vector_add_i32", data_in_ref=(ta, tb), data_out_ref=to))
    np.testing.assert_array_equal(to.cpu().numpy(), W.vector_add_i32(a, b))
    with pytest.raises(ConfigError):
        WorkDescriptor(slot=61, kind="vector_add_i32", data_in_ref=(ta.float(), tb), data_out_ref=to).to_c()
