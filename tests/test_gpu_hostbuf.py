"""Zero-copy payloads in mapped pinned host memory (HostBuffer, LK_DF_HOSTMEM)
against the numpy oracle -- the B200 replacement for the reference's
Copyin/Copyout phases (P/host.py:212-224) on small transfers.

Bars as in test_gpu_payload.py: integer and SAXPY bit-exact, reduce bit-exact
against oracle/work.py's fixed order.  The staleness tests rewrite the host
inputs in place between dispatches of one staged (cached) slot: a worker that
read them through a GPU cache line left by the previous dispatch would return
the old result.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import work as W
from paper_2310_01212_b200 import host, native
from paper_2310_01212_b200.device import DeviceBuffer, HostBuffer, WorkDescriptor, reduce_blocks
from paper_2310_01212_b200.errors import UsageError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["direct", "gateway"])
def session(request):
    s, _ = native.NativeSession.start(native.NativeConfig(num_workers=None, spin_yield_threshold=200,
                                                          poll_mode=request.param, record_trace=True,
                                                          trace_capacity=4096))
    yield s
    s.close()


def _i32(n, seed):
    return np.random.default_rng(seed).integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)


def _f32(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n).astype(np.float32)


def run(s, mask, work):
    s.trigger(mask, work)
    s.wait(mask)


MASKS = {"one": lambda n: 1, "four": lambda n: 0b1111, "all": lambda n: host.full_mask(n)}


@pytest.mark.parametrize("mask_name", list(MASKS))
@pytest.mark.parametrize("n", [1, 3, 4, 1000, 4097, 65536])
def test_vector_add_host_in_host_out(session, mask_name, n):
    a, b = _i32(n, 0), _i32(n, 1)
    ha, hb, ho = HostBuffer.from_array(a), HostBuffer.from_array(b), HostBuffer(4 * n)
    run(session, MASKS[mask_name](session.num_workers),
        WorkDescriptor(slot=40, kind="vector_add_i32", data_in_ref=(ha, hb), data_out_ref=ho))
    np.testing.assert_array_equal(ho.array(np.int32, n), W.vector_add_i32(a, b))


@pytest.mark.parametrize("n", [5, 4096, 100_003])
def test_saxpy_mixed_host_and_device(session, n):
    x, y = _f32(n, 2), _f32(n, 3)
    hx, dy, ho = HostBuffer.from_array(x), DeviceBuffer.from_array(y), HostBuffer(4 * n)
    run(session, 0b1011, WorkDescriptor(slot=41, kind="saxpy_f32", data_in_ref=(hx, dy), data_out_ref=ho,
                                        alpha=1.5))
    np.testing.assert_array_equal(ho.array(np.float32, n), W.saxpy_f32(1.5, x, y))


@pytest.mark.parametrize("direction", ["h2d", "d2h"])
def test_hbm_stream_across_the_link(session, direction):
    n = 12_345
    src = _i32(n, 4)
    if direction == "h2d":
        s_buf, d_buf = HostBuffer.from_array(src), DeviceBuffer(4 * n)
    else:
        s_buf, d_buf = DeviceBuffer.from_array(src), HostBuffer(4 * n)
    run(session, 0b11, WorkDescriptor(slot=42, kind="hbm_stream", data_in_ref=s_buf, data_out_ref=d_buf))
    np.testing.assert_array_equal(d_buf.download(np.int32, n), W.hbm_stream(src))


@pytest.mark.parametrize("n", [7, 4096, 70_001])
def test_reduce_host_input_host_total(session, n):
    x = _f32(n, 5)
    hx, dp, ht = HostBuffer.from_array(x), DeviceBuffer(8 * reduce_blocks(n)), HostBuffer(8)
    run(session, 0b111, WorkDescriptor(slot=43, kind="block_reduce_f32", data_in_ref=hx, data_out_ref=dp,
                                       total_ref=ht))
    parts = dp.download(np.float64, reduce_blocks(n))
    np.testing.assert_array_equal(parts.view(np.uint64), W.block_reduce_partials(x).view(np.uint64))
    assert np.float64(ht.array(np.float64, 1)[0]).view(np.uint64) == \
        np.float64(W.block_reduce_total(x)).view(np.uint64)


@pytest.mark.parametrize("mask_name", ["one", "all"])
def test_host_rewrite_between_cached_dispatches(session, mask_name):
    """One staged slot re-triggered 40 times (the cached-descriptor fast
    path); the host rewrites both inputs in place before every trigger and
    reads the output after every wait."""
    n = 3000
    ha, hb, ho = HostBuffer(4 * n), HostBuffer(4 * n), HostBuffer(4 * n)
    work = WorkDescriptor(slot=44, kind="vector_add_i32", data_in_ref=(ha, hb), data_out_ref=ho)
    mask = MASKS[mask_name](session.num_workers)
    va, vb, vo = ha.array(np.int32), hb.array(np.int32), ho.array(np.int32)
    for k in range(40):
        a, b = _i32(n, 100 + k), _i32(n, 200 + k)
        va[:] = a
        vb[:] = b
        run(session, mask, work)
        np.testing.assert_array_equal(vo, W.vector_add_i32(a, b), err_msg=f"dispatch {k}")


def test_single_word_round_trip_sees_every_host_value(session):
    """The paper's small-transfer case at its smallest: a
    4-byte input and output, one worker, 500 values in a row."""
    ha, hb, ho = HostBuffer(4), HostBuffer(4), HostBuffer(4)
    work = WorkDescriptor(slot=45, kind="vector_add_i32", data_in_ref=(ha, hb), data_out_ref=ho)
    va, vb, vo = ha.array(np.int32), hb.array(np.int32), ho.array(np.int32)
    vb[0] = 1
    for k in range(500):
        va[0] = k
        run(session, 1 << (k % 3), work)
        assert vo[0] == k + 1


def test_trace_of_host_buffer_session_validates(session):
    from oracle import protocol as O
    ha, hb, ho = HostBuffer(64), HostBuffer(64), HostBuffer(64)
    run(session, 0b1, WorkDescriptor(slot=46, kind="vector_add_i32", data_in_ref=(ha, hb), data_out_ref=ho))
    writes = [(r.side, r.sm_id, r.word) for r in session.recorded_trace()]
    assert O.replay(writes).violation is None


def test_reduce_partials_in_host_memory_refused(session):
    x = HostBuffer(4 * 4096)
    with pytest.raises(UsageError, match="partials"):
        session.trigger(1, WorkDescriptor(slot=47, kind="block_reduce_f32", data_in_ref=x,
                                          data_out_ref=HostBuffer(8)))
    run(session, 1, WorkDescriptor(slot=47, kind="empty"))     # the session is unharmed


def test_unregistered_host_address_refused(session):
    a = np.zeros(1024, np.int32)
    with pytest.raises(UsageError, match="neither device memory nor mapped pinned host memory"):
        session.trigger(1, WorkDescriptor(slot=48, kind="hbm_stream", data_in_ref=int(a.ctypes.data), n=1024,
                                          data_out_ref=DeviceBuffer(4096)))
    run(session, 1, WorkDescriptor(slot=48, kind="empty"))


def test_alloc_and_free_while_resident(session):
    """cudaFreeHost synchronizes the device; a pinned free while the
    persistent kernel is resident is deferred (it would otherwise wait on the
    kernel forever), and allocation does not wait at all."""
    for _ in range(5):
        b = HostBuffer(1 << 16)
        b.array(np.int32)[:] = 7
        b.free()
    run(session, 1, WorkDescriptor(slot=49, kind="empty"))


@pytest.mark.parametrize("kind", ["vector_add_i32", "saxpy_f32", "hbm_stream"])
@pytest.mark.parametrize("where", ["device", "host"])
def test_empty_payloads_complete_and_touch_nothing(session, kind, where):
    """n = 0 on every worker (an empty input is legal in the reference's
    descriptors): the handshake completes, the output guard words are left
    alone, and the session keeps working."""
    cls = HostBuffer if where == "host" else DeviceBuffer
    guard = np.full(4, 0x5A5A5A5A, np.int32)
    a, b, o = cls.from_array(guard), cls.from_array(guard), cls.from_array(guard)
    ins = (a,) if kind == "hbm_stream" else (a, b)
    run(session, host.full_mask(session.num_workers),
        WorkDescriptor(slot=50, kind=kind, data_in_ref=ins if len(ins) > 1 else ins[0], data_out_ref=o, n=0))
    np.testing.assert_array_equal(o.download(np.int32, 4), guard)
    run(session, 1, WorkDescriptor(slot=51, kind="empty"))


def test_pinned_torch_tensors_are_zero_copy_payloads(session):
    """torch CPU tensors in pinned memory (cudaHostAlloc under UVA: mapped,
    device address = host address) are accepted as zero-copy payload refs
    like HostBuffers; pageable CPU tensors are refused."""
    torch = pytest.importorskip("torch")
    n = 10_001
    a = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32).pin_memory()
    b = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32).pin_memory()
    o = torch.empty(n, dtype=torch.int32).pin_memory()
    run(session, 0b111, WorkDescriptor(slot=52, kind="vector_add_i32", data_in_ref=(a, b), data_out_ref=o))
    np.testing.assert_array_equal(o.numpy(), W.vector_add_i32(a.numpy(), b.numpy()))
    with pytest.raises(UsageError, match="pinned host memory"):
        WorkDescriptor(slot=53, kind="vector_add_i32", data_in_ref=(torch.zeros(4, dtype=torch.int32),) * 2,
                       data_out_ref=o).to_c()
