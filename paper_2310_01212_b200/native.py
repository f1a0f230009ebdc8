"""The B200 persistent-worker session: drop-in for persistkern.native.

``NativeSession`` keeps the reference's API
(/root/reference/pkg/src/persistkern/native.py:82-299: ``start`` / ``trigger`` /
``wait`` / ``dispose`` / ``recorded_trace``, the ``to_gpu`` / ``from_gpu`` /
``worker_phase`` views, ``_spin_until``) but its workers are the CTAs of one
resident sm_100a kernel, one per SM, and its mailboxes are pinned mapped host
words.  Every call goes straight to liblk.so (include/lk.h) with the GIL
released; there is no Python or CPU execution path behind it.

``LaunchSyncBaseline`` is the conventional flow the paper compares against
(``ThreadSpawnBaseline``, native.py:304-331): one cudaLaunchKernel of the same
work function per task, then cudaStreamSynchronize.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import logging
import time
import weakref
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib, protocol
from .device import WorkDescriptor, as_work
from .errors import HangDetected, UsageError
from .host import (PHASE_COPYIN, PHASE_COPYOUT, PHASE_DISPOSE, PHASE_INIT, PHASE_LAUNCH,
                   PHASE_TRIGGER, PHASE_WAIT, PhaseTiming, TimingLog, _check_mask, full_mask, sms_in_mask)

log = logging.getLogger(__name__)

PURE_SPIN = "pure_spin"
SPIN_THEN_YIELD = "spin_then_yield"
BACKEND = "b200"
POLL_MODES = {"direct": _lib.POLL_DIRECT, "gateway": _lib.POLL_GATEWAY, "hybrid": _lib.POLL_HYBRID}


@dataclass(frozen=True)
class NativeConfig:
    """Session configuration (reference fields first, native.py:44-60).

    ``num_workers`` defaults to 4 like the reference's (native.py:46);
    ``num_workers=None`` means one worker per SM (148 on B200).  The spin
    settings govern the *host* spin in lk_wait; device workers always spin in
    hardware, optionally backing off with ``poll_backoff_ns`` of __nanosleep.
    """

    num_workers: Optional[int] = 4
    pin_to_cores: bool = False
    spin_strategy: str = SPIN_THEN_YIELD
    spin_yield_threshold: int = 10_000
    busy_loop_ns_per_iteration: float = 25.0
    record_trace: bool = False
    wait_timeout_s: float = 10.0
    # B200 knobs
    device: int = 0
    threads_per_worker: int = 512
    poll_backoff_ns: int = 0
    cell_stride: int = 128          # bytes between to_gpu cells
    status_stride: int = 32         # bytes between from_gpu status cells (32: two workers per host line)
    poll_mode: str = "direct"       # "direct": each worker polls its host cell; "gateway": one warp
                                    # polls all host cells and forwards through device memory
    poll_replicas: int = 1          # one to_gpu cell per worker (replicas were measured slower and removed)
    poll_spacing_ns: int = 300
    num_slots: int = 1024
    trace_capacity: int = 65536
    acquire_poll: bool = True       # polls are ld.acquire.sys (False: relaxed; tools/ab_acquire.py)
    fence_always: bool = False
    tma_payload: bool = True        # payload tiles via the TMA bulk ring (False: 128-bit LSU loads)
    ring_stages: int = 6            # TMA ring depth, 16-KiB stages (2..12)
    sm_partition: int = 0           # N > 0: run in a green context of >= N SMs (multiple of 8), one
                                    # worker per partition SM; the rest stay free for other kernels
    timeline: bool = False          # gateway forward stamps in last_timeline() (one extra L2 load)
    ack_delay_ns: int = 300         # direct/1 replica: first poll for the ack this long after FINISHED (0: at
                                    # once); adapted per worker to the host's answer time
    ack_adaptive: bool = True       # False: keep ack_delay_ns fixed
    idle_delay_ns: int = 0          # first poll for the next WORK this long after the closing NOP (start;
                                    # adapted up for back-to-back re-triggers of one worker)
    tma_min_workers: int = 49       # payload dispatches to fewer workers use LSU loads (1: always the ring)
    lazy_ack: bool = False          # wait() returns once the ack is written; its consumption is
                                    # awaited by the next trigger/dispose of that worker
    host_descriptors: bool = False  # descriptor table in pinned mapped host memory (direct mode):
                                    # trigger/wait/register make no CUDA call, so the session works
                                    # while a serialising profiler (ncu) holds the kernel's launch
    full_board: bool = False        # direct mode: every mailbox write ships the whole board (the
                                    # paper's workaround for deferred small transfers)

    def __post_init__(self) -> None:
        if self.num_workers is not None and self.num_workers < 1:
            raise UsageError("num_workers must be >= 1")
        if self.spin_strategy not in (PURE_SPIN, SPIN_THEN_YIELD):
            raise UsageError(f"unknown spin strategy {self.spin_strategy!r}")
        if self.spin_strategy == SPIN_THEN_YIELD and self.spin_yield_threshold <= 0:
            raise UsageError("spin_yield_threshold must be positive")
        if self.wait_timeout_s <= 0:
            raise UsageError("wait_timeout_s must be positive")
        if self.poll_mode not in POLL_MODES:
            raise UsageError(f"unknown poll mode {self.poll_mode!r}")
        if not 0 <= self.ack_delay_ns <= 100_000 or not 0 <= self.idle_delay_ns <= 100_000:
            raise UsageError("ack_delay_ns and idle_delay_ns must be in [0, 100000]")
        if self.tma_min_workers < 1:
            raise UsageError("tma_min_workers must be >= 1")

    def to_c(self) -> "_lib.lk_config":
        c = _lib.lk_config()
        c.num_workers = self.num_workers or 0
        c.threads_per_worker = self.threads_per_worker
        c.device = self.device
        c.spin_strategy = 0 if self.spin_strategy == PURE_SPIN else 1
        c.spin_yield_threshold = self.spin_yield_threshold
        c.record_trace = 1 if self.record_trace else 0
        c.trace_capacity = self.trace_capacity
        c.poll_backoff_ns = self.poll_backoff_ns
        c.cell_stride = self.cell_stride
        c.status_stride = self.status_stride
        c.ring_stages = self.ring_stages
        c.sm_partition = self.sm_partition
        c.num_slots = self.num_slots
        c.poll_replicas = self.poll_replicas
        c.poll_spacing_ns = self.poll_spacing_ns
        c.poll_mode = POLL_MODES[self.poll_mode]
        c.wait_timeout_ns = int(self.wait_timeout_s * 1e9)
        c.ack_delay_ns = self.ack_delay_ns
        c.idle_delay_ns = self.idle_delay_ns
        c.tma_min_workers = self.tma_min_workers
        c.flags = ((_lib.CF_ACQUIRE_POLL if self.acquire_poll else _lib.CF_RELAXED_POLL)
                   | (_lib.CF_FENCE_ALWAYS if self.fence_always else 0)
                   | (0 if self.tma_payload else _lib.CF_LSU_PAYLOAD)
                   | (_lib.CF_TIMELINE if self.timeline else 0)
                   | (_lib.CF_LAZY_ACK if self.lazy_ack else 0)
                   | (0 if self.ack_delay_ns else _lib.CF_NO_ACK_DELAY)
                   | (0 if self.ack_adaptive else _lib.CF_ACK_FIXED)
                   | (_lib.CF_HOST_DESC if self.host_descriptors else 0)
                   | (_lib.CF_FULL_BOARD if self.full_board else 0))
        return c


def init_device(device: int = 0) -> None:
    """Create the device's primary CUDA context now (a one-byte allocation
    through liblk.so), so the driver's helper threads are spawned with the
    caller's current CPU affinity rather than a later, narrower one."""
    lib = _lib.load()
    p = C.c_uint64()
    _lib.check(lib.lk_dev_alloc(device, 1, C.byref(p)))
    _lib.check(lib.lk_dev_free(p.value))


def device_count() -> int:
    """Visible CUDA devices (lk_device_count); 0 without a GPU."""
    n = C.c_int()
    return n.value if _lib.load().lk_device_count(C.byref(n)) == 0 else 0


def under_profiler() -> bool:
    """True inside a CUDA tool that injects itself into the process: Nsight
    Compute's launcher exports NV_TPS_LAUNCH_TOKEN and the
    NV_NSIGHT_INJECTION_* / NV_COMPUTE_PROFILER_PERFWORKS_DIR variables
    (seen on the B200 box), other injection tools CUDA_INJECTION64_PATH.
    Such tools may serialise launches, so a live session must then make no
    CUDA calls."""
    import os
    keys = ("NV_TPS_LAUNCH_TOKEN", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE", "NV_COMPUTE_PROFILER_PERFWORKS_DIR",
            "CUDA_INJECTION64_PATH")
    return any(os.environ.get(k) for k in keys)


def pin_host_thread(device: int) -> int:
    """Pin the calling thread to the GPU's NUMA-local cores; returns core count."""
    n = C.c_uint32()
    _lib.check(_lib.load().lk_pin_thread_near(device, C.byref(n)))
    return n.value


_LAZY_WARNED = False


def _timing(phase: str, ns: int, mask: int) -> PhaseTiming:
    """PhaseTiming for a validated phase/mask without re-running __post_init__
    (the checks hold by construction here: ns >= 0, mask > 0)."""
    t = _new(PhaseTiming)
    t.__dict__.update(phase=phase, cycles=ns, sm_mask=mask)
    return t


_new = object.__new__


def _make_fast(session: "NativeSession", raw):
    """The CPython fast path (csrc/lk_pyfast.c) bound to this session, or
    None when the module was not built (the ctypes calls then serve every
    call; both go to liblk.so)."""
    try:
        from . import _lkfast
    except ImportError:
        log.debug("_lkfast not built: trigger/wait use ctypes only")
        return None
    addr = lambda fn: C.cast(fn, C.c_void_p).value  # noqa: E731
    # keep_gil=False: lk_trigger drops the GIL like every other call.  Holding
    # it across the ~100-ns call measured within noise (tools/ab_gil.py)
    # and would stall other Python threads if the call ever spun.
    keep_gil = False
    # declines go to the session's Python path (held weakly: the session owns
    # the Fast object through its bound methods), errors to _raise_lk
    return _lkfast.Fast(session._h.value, session.nwords, addr(raw.lk_trigger), addr(raw.lk_wait),
                        session._staged, session._mask_cache, session._timings._rows,
                        1 << session.num_workers, PhaseTiming, WorkDescriptor, PHASE_TRIGGER, PHASE_WAIT, keep_gil,
                        NativeSession._trigger_slow, NativeSession._wait_slow, weakref.ref(session), _raise_lk)


def _raise_lk(rc: int, mask: int, is_wait: int) -> None:
    """Raise the exception of an LK_E_* code from the fast path (as the Python
    path would: a wait names its workers)."""
    if is_wait:
        _lib.raise_for(rc, sm_ids=tuple(sms_in_mask(mask)))
    _lib.raise_for(rc)


def _warn_lazy_loading() -> None:
    """CUDA 12 loads kernel modules lazily on first launch, and a module load
    while the persistent kernel is resident can wait on it forever.  liblk.so
    preloads its own kernels; other libraries' kernels (torch ...) must be
    launched once before start(), or CUDA_MODULE_LOADING=EAGER set."""
    global _LAZY_WARNED
    import os
    import sys
    if _LAZY_WARNED or os.environ.get("CUDA_MODULE_LOADING", "LAZY").upper() == "EAGER":
        return
    if "torch" in sys.modules:
        _LAZY_WARNED = True
        log.info("CUDA lazy module loading is on: launch every torch kernel you will use while "
                 "the LK session is live once before start() (or set CUDA_MODULE_LOADING=EAGER)")


class _WorkerHandle:
    """Stands in for the reference's per-worker threading.Thread."""

    def __init__(self, session: "NativeSession", wid: int):
        self._s, self.wid = session, wid
        self.name = f"lk-worker-{wid}"

    def is_alive(self) -> bool:
        return self._s._kernel_alive() and self._s.worker_phase[self.wid] is not protocol.Phase.EXITED


class NativeSession:
    """A booted persistent kernel (one CTA per SM) plus its mailboard."""

    def __init__(self, cfg: NativeConfig, handle: C.c_void_p, num_workers: int):
        self.cfg = cfg
        self._lib = _lib.load()
        raw = _lib.raw()
        self._raw_trigger, self._raw_wait = raw.lk_trigger, raw.lk_wait   # hot path: no argtypes
        self._h = handle
        self.num_workers = num_workers
        self.nwords = (num_workers + 63) // 64
        self.disposed = False
        self.timings = TimingLog()   # a list[PhaseTiming] (host.TimingLog)
        self.descriptors: dict[int, WorkDescriptor] = {}
        self._staged: dict[int, tuple] = {}
        self._threads = [_WorkerHandle(self, i) for i in range(num_workers)]
        self._u64 = C.c_uint64()
        self._u64_ref = C.byref(self._u64)
        self._mask_cache: dict[int, bytes] = {}
        self._cells = (C.c_uint32 * num_workers)()
        self._cells2 = (C.c_uint32 * num_workers)()
        self._cells3 = (C.c_uint32 * num_workers)()
        self._raw = raw
        self._fast = None
        self._bind_fast()

    # -- bring-up ----------------------------------------------------------

    @classmethod
    def start(cls, cfg: Optional[NativeConfig] = None) -> tuple["NativeSession", PhaseTiming]:
        cfg = cfg or NativeConfig()   # the reference's default: 4 workers
        lib = _lib.load()
        _warn_lazy_loading()
        t0 = time.perf_counter_ns()
        if cfg.pin_to_cores:
            try:
                pin_host_thread(cfg.device)
            except Exception as exc:   # downgrade like _maybe_pin (native.py:70-79)
                log.warning("host core pinning failed (%s); running unpinned", exc)
        h = C.c_void_p()
        init_ns = C.c_uint64()
        _lib.check(lib.lk_create(C.byref(cfg.to_c()), C.byref(h), C.byref(init_ns)))
        n = C.c_uint32()
        _lib.check(lib.lk_num_workers(h, C.byref(n)))
        if cfg.num_workers is None:
            cfg = dataclasses.replace(cfg, num_workers=n.value)
        session = cls(cfg, h, n.value)
        timing = PhaseTiming(PHASE_INIT, time.perf_counter_ns() - t0, full_mask(n.value))
        session.timings.append(timing)
        return session, timing

    # -- views of the mailboard (native.py:88-94) --------------------------

    def _read_cells(self):
        _lib.check(self._lib.lk_read_cells(self._h, self._cells, self._cells2, self._cells3,
                                           self.num_workers))
        return list(self._cells), list(self._cells2), list(self._cells3)

    @property
    def to_gpu(self) -> list[int]:
        return self._read_cells()[0]

    @property
    def from_gpu(self) -> list[int]:
        return self._read_cells()[1]

    @property
    def worker_phase(self) -> list[protocol.Phase]:
        return [protocol.PHASE_OF_CODE[c] for c in self._read_cells()[2]]

    @property
    def worker_error(self) -> list[Optional[BaseException]]:
        out: list[Optional[BaseException]] = []
        code, word = C.c_uint32(), C.c_uint32()
        for i in range(self.num_workers):
            _lib.check(self._lib.lk_worker_error(self._h, i, C.byref(code), C.byref(word)))
            out.append(None if code.value == 0 else protocol.ProtocolViolation(
                f"{_lib.WERR_NAMES.get(code.value, 'device error')} (word {word.value})",
                word=word.value))
        return out

    @property
    def pending_mask(self) -> int:
        buf = (C.c_uint64 * self.nwords)()
        _lib.check(self._lib.lk_pending(self._h, buf, self.nwords))
        return int.from_bytes(bytes(buf), "little")

    @property
    def partition_info(self) -> tuple[int, int]:
        """(SMs of this session's green-context partition, SMs left for other
        kernels); (0, 0) when the session spans the GPU."""
        a, b = C.c_uint32(), C.c_uint32()
        _lib.check(self._lib.lk_partition_info(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    @property
    def smid_map(self) -> list[int]:
        """%smid of each worker's CTA: the B200 form of check_block_mapping."""
        buf = (C.c_uint32 * self.num_workers)()
        _lib.check(self._lib.lk_smid_map(self._h, buf, self.num_workers))
        return list(buf)

    def _kernel_alive(self) -> bool:
        a = C.c_uint32()
        _lib.check(self._lib.lk_kernel_alive(self._h, C.byref(a)))
        return bool(a.value)

    # -- host side -----------------------------------------------------------

    @property
    def timings(self) -> TimingLog:
        """Every PhaseTiming of this session, in order (a list, P/native.py:99)."""
        return self._timings

    @timings.setter
    def timings(self, v) -> None:
        # callers may rebind it (session.timings = []): keep the TimingLog
        # type and point the C fast path at the new rows
        self._timings = v if isinstance(v, TimingLog) else TimingLog(v)
        if getattr(self, "_fast", None) is not None:
            self._bind_fast()

    def _bind_fast(self) -> None:
        """Serve `trigger`/`wait` from the CPython fast path: its methods become
        this session's own attributes, so the common call runs no Python frame."""
        self._fast = f = _make_fast(self, self._raw)
        if f is not None:
            self.__dict__["trigger"] = f.trigger
            self.__dict__["wait"] = f.wait

    def _unbind_fast(self) -> None:
        if self._fast is not None:
            self._fast.close()   # method objects captured earlier stop calling into liblk.so
        self._fast = None
        self.__dict__.pop("trigger", None)
        self.__dict__.pop("wait", None)

    def _require_live(self) -> None:
        if self.disposed:
            raise UsageError("session already disposed")

    def _check(self, mask: int) -> None:
        # host._check_mask's rules (host.py:76-81) without building the id list:
        # a 148-bit mask would otherwise cost ~30 us of Python per call
        if mask <= 0 or mask >> self.num_workers:
            _check_mask(mask, self.num_workers)   # raises with the reference's message

    def _mask(self, mask: int) -> bytes:
        b = self._mask_cache.get(mask)
        if b is None:
            if len(self._mask_cache) > 4096:
                self._mask_cache.clear()
            b = self._mask_cache[mask] = mask.to_bytes(8 * self.nwords, "little")
        return b

    def register(self, work: WorkDescriptor, mask: int = 0) -> int:
        """Stage ``work`` in its device slot (a no-op when already staged).

        Returns the ns spent.  Payload kinds record the worker set that will
        shard them, so a new mask for the same descriptor re-stages it.
        """
        t0 = time.perf_counter_ns()
        work = as_work(work)
        key = mask if work.multi_worker else 0
        if self._is_staged(work, key):
            return 0   # same descriptor object already staged with this mask
        d = work.to_c()
        rc = self._lib.lk_register_desc(self._h, work.slot, C.byref(d), self._mask(key), self.nwords)
        _lib.check(rc)
        self.descriptors[work.slot] = work
        self._staged[work.slot] = (work, key, work.multi_worker)
        return time.perf_counter_ns() - t0

    # trigger and wait are the per-task hot path: the helpers (_check, _mask,
    # _is_staged, _timing) are inlined, which halves the wrapper's cost over
    # the bare ctypes calls (tools/py_overhead.py).  Semantics are the helpers'.
    def trigger(self, mask: int, work: WorkDescriptor) -> PhaseTiming:
        """Dispatch: one word write per masked worker, no kernel launch.

        A live session normally answers this name from its instance: the
        CPython fast path (csrc/lk_pyfast.c), which hands anything it does not
        serve to _trigger_slow.  This method serves explicit class calls."""
        f = self._fast
        if f is not None:
            return f.trigger(mask, work)
        return self._trigger_slow(mask, work)

    def _trigger_slow(self, mask: int, work: WorkDescriptor) -> PhaseTiming:
        if self.disposed:
            raise UsageError("session already disposed")
        if mask <= 0 or mask >> self.num_workers:
            _check_mask(mask, self.num_workers)   # raises with the reference's message
        if type(work) is not WorkDescriptor:
            work = as_work(work)
        slot = work.slot
        # identity, not dataclass equality: two descriptors with equal fields
        # may point at different buffers (their refs are compare=False)
        st = self._staged.get(slot)
        if st is not None and st[0] is work and st[1] == (mask if st[2] else 0):
            d = None   # this descriptor object is already staged for this worker set
        else:
            d = C.byref(work.to_c())
        b = self._mask_cache.get(mask)
        if b is None:
            b = self._mask(mask)
        trig = self._raw_trigger if slot <= 0x7FFFFFFF else self._lib.lk_trigger   # raw: C int args
        rc = trig(self._h, b, self.nwords, slot, d, self._u64_ref)
        if rc:
            _lib.raise_for(rc)
        if d is not None:
            multi = work.multi_worker
            self.descriptors[slot] = work
            self._staged[slot] = (work, mask if multi else 0, multi)
        row = (PHASE_TRIGGER, self._u64.value, mask)
        self._timings._rows.append(row)
        t = _new(PhaseTiming)
        td = t.__dict__
        td["phase"], td["cycles"], td["sm_mask"] = row
        return t

    def _is_staged(self, work: WorkDescriptor, key: int) -> bool:
        st = self._staged.get(work.slot)
        return st is not None and st[0] is work and st[1] == key

    def wait(self, mask: int) -> PhaseTiming:
        """Spin (in C) until every masked worker published FINISHED, then ack.
        (Served like trigger: the fast path, falling back to _wait_slow.)"""
        f = self._fast
        if f is not None:
            return f.wait(mask)
        return self._wait_slow(mask)

    def _wait_slow(self, mask: int) -> PhaseTiming:
        if self.disposed:
            raise UsageError("session already disposed")
        if mask <= 0 or mask >> self.num_workers:
            _check_mask(mask, self.num_workers)
        b = self._mask_cache.get(mask)
        if b is None:
            b = self._mask(mask)
        rc = self._raw_wait(self._h, b, self.nwords, self._u64_ref)
        if rc:
            _lib.raise_for(rc, sm_ids=tuple(sms_in_mask(mask)))
        row = (PHASE_WAIT, self._u64.value, mask)
        self._timings._rows.append(row)
        t = _new(PhaseTiming)
        td = t.__dict__
        td["phase"], td["cycles"], td["sm_mask"] = row
        return t

    def _spin_until(self, cond, what: str, sm_ids) -> int:
        """Python-level poll helper with the reference's timeout contract."""
        deadline = time.monotonic() + self.cfg.wait_timeout_s
        while True:
            if cond():
                return time.perf_counter_ns()
            if time.monotonic() > deadline:
                raise HangDetected(f"{what} made no progress within {self.cfg.wait_timeout_s}s",
                                   sm_ids=tuple(sm_ids))
            time.sleep(0)

    def copyin(self, buf, host_array: np.ndarray) -> PhaseTiming:
        """Stage a payload host->device (Copyin phase, host.py:212-213)."""
        t0 = time.perf_counter_ns()
        a = np.ascontiguousarray(host_array)
        _lib.check(self._lib.lk_memcpy_h2d(_dev_addr(buf), a.ctypes.data, a.nbytes))
        timing = PhaseTiming(PHASE_COPYIN, time.perf_counter_ns() - t0)
        self.timings.append(timing)
        return timing

    def copyout(self, host_array: np.ndarray, buf) -> PhaseTiming:
        """Read a result device->host (Copyout phase, host.py:215-216)."""
        t0 = time.perf_counter_ns()
        _lib.check(self._lib.lk_memcpy_d2h(host_array.ctypes.data, _dev_addr(buf), host_array.nbytes))
        timing = PhaseTiming(PHASE_COPYOUT, time.perf_counter_ns() - t0)
        self.timings.append(timing)
        return timing

    def dispose(self) -> PhaseTiming:
        """EXIT to every worker; the persistent kernel retires."""
        self._require_live()
        rc = self._lib.lk_dispose(self._h, C.byref(self._u64))
        _lib.check(rc, sm_ids=tuple(range(self.num_workers)))
        self.disposed = True
        self._unbind_fast()
        timing = PhaseTiming(PHASE_DISPOSE, self._u64.value, full_mask(self.num_workers))
        self.timings.append(timing)
        return timing

    def abort(self, timeout_s: float = 10.0) -> None:
        """Retire the kernel whatever the host state (dead worker, pending work)."""
        if self._h:
            self._unbind_fast()
            _lib.check(self._lib.lk_abort(self._h, int(timeout_s * 1e9)))
            self.disposed = True

    def close(self) -> None:
        """Dispose (or abort) if needed and free the runtime's memory."""
        self._unbind_fast()
        if self._h:
            if not self.disposed:
                try:
                    self.dispose()
                except Exception:
                    self.abort()
            self._lib.lk_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            if self._h and self.disposed:
                self._lib.lk_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # -- tracing ----------------------------------------------------------------

    def trace_arrays(self):
        """The linearized trace as numpy arrays (step, side, worker, word, hseq, t_ns)."""
        n = C.c_uint64()
        _lib.check(self._lib.lk_trace_count(self._h, C.byref(n)))
        buf = (_lib.lk_trace_rec * max(1, n.value))()
        _lib.check(self._lib.lk_trace_read(self._h, buf, n.value, C.byref(n)))
        dt = np.dtype([("step", "<u8"), ("side", "<u4"), ("worker", "<u4"), ("word", "<u4"),
                       ("hseq", "<u4"), ("t_ns", "<u8")])
        return np.frombuffer(bytes(buf), dtype=dt, count=n.value).copy()

    def recorded_trace(self) -> list[protocol.TraceRecord]:
        """Records in linearized order (per-worker causal order is exact)."""
        a = self.trace_arrays()
        return [protocol.TraceRecord(int(r["step"]), chr(r["side"]), int(r["worker"]), int(r["word"]))
                for r in a]

    # -- measurement ------------------------------------------------------------

    def bench_roundtrip(self, masks: list[int], slot: int, rounds: int):
        """Closed-loop trigger+wait rounds run entirely in C.

        Returns (trigger_ns, done_ns, cycle_ns) numpy arrays: trigger call,
        trigger start -> last FINISHED seen, trigger start -> ack consumed.
        """
        packed = b"".join(self._mask(m) for m in masks)
        trig = np.zeros(rounds, dtype=np.uint64)
        done = np.zeros(rounds, dtype=np.uint64)
        cyc = np.zeros(rounds, dtype=np.uint64)
        rc = self._lib.lk_bench_roundtrip(self._h, packed, len(masks), self.nwords, slot, rounds,
                                          trig.ctypes.data, done.ctypes.data, cyc.ctypes.data)
        _lib.check(rc)
        return trig, done, cyc

    def bench_roundtrip_gaps(self, masks: list[int], slot: int, rounds: int):
        """bench_roundtrip plus, per round, the largest gap (ns) in the host
        thread's own spin loop (lk_bench_roundtrip_gaps): rounds whose gap is
        microseconds long were slowed by the host thread being descheduled."""
        packed = b"".join(self._mask(m) for m in masks)
        trig = np.zeros(rounds, dtype=np.uint64)
        done = np.zeros(rounds, dtype=np.uint64)
        cyc = np.zeros(rounds, dtype=np.uint64)
        gap = np.zeros(rounds, dtype=np.uint64)
        rc = self._lib.lk_bench_roundtrip_gaps(self._h, packed, len(masks), self.nwords, slot, rounds,
                                               trig.ctypes.data, done.ctypes.data, cyc.ctypes.data,
                                               gap.ctypes.data)
        _lib.check(rc)
        return trig, done, cyc, gap

    def last_timeline(self) -> np.ndarray:
        """(num_workers, 8) record of each worker's last dispatch: globaltimer ns
        at value seen, work begin, work end, FINISHED issued, gateway forward
        (timeline=True); clock64 at value seen, work begin, FINISHED issued."""
        t = np.zeros((self.num_workers, 16), dtype=np.uint64)
        _lib.check(self._lib.lk_last_timeline(self._h, t.ctypes.data, self.num_workers))
        return t

    def fast_counts(self) -> np.ndarray:
        """Per-worker count of to_gpu values the kernel's fast path settled
        since boot (lk_fast_count): IDLE x WORK of an empty or cached
        single-thread item, IDLE x WORK begin of a payload item, FINISHED x NOP."""
        c = np.zeros(self.num_workers, dtype=np.uint32)
        _lib.check(self._lib.lk_fast_count(self._h, c.ctypes.data, self.num_workers))
        return c

    def last_host_times(self) -> np.ndarray:
        """(num_workers, 3) CLOCK_MONOTONIC ns of each worker's last dispatch:
        trigger start, WORK written, FINISHED observed."""
        t = np.zeros((self.num_workers, 3), dtype=np.uint64)
        _lib.check(self._lib.lk_last_host_times(self._h, t.ctypes.data, self.num_workers))
        return t

    def last_spans(self):
        """Device globaltimer (begin, end) of each worker's last dispatch."""
        b = np.zeros(self.num_workers, dtype=np.uint64)
        e = np.zeros(self.num_workers, dtype=np.uint64)
        _lib.check(self._lib.lk_last_spans(self._h, b.ctypes.data, e.ctypes.data, self.num_workers))
        return b, e


def _dev_addr(buf) -> int:
    from .device import _addr
    return _addr(buf)


class LaunchSyncBaseline:
    """cudaLaunchKernel + cudaStreamSynchronize per task (the CUDA "spawn")."""

    def __init__(self, device: int = 0, threads_per_worker: int = 512, grid: Optional[int] = None,
                 tma_payload: bool = True, beside: Optional["NativeSession"] = None):
        """``beside``: a session started with ``sm_partition``; the baseline's
        kernels then run on the SMs that session left free, concurrently with it."""
        self._lib = _lib.load()
        self._h = C.c_void_p()
        if beside is not None:
            _lib.check(self._lib.lk_baseline_create_in(beside._h, threads_per_worker, C.byref(self._h)))
        else:
            _lib.check(self._lib.lk_baseline_create(device, threads_per_worker, C.byref(self._h)))
        _lib.check(self._lib.lk_baseline_set_tma(self._h, 1 if tma_payload else 0))
        if grid is None:
            if beside is not None:
                grid = beside.partition_info[1]
            else:
                n = C.c_int()
                _lib.check(self._lib.lk_sm_count(device, C.byref(n)))
                grid = n.value
        self.grid = grid
        self.timings = TimingLog()   # a list[PhaseTiming] (host.TimingLog)
        self._u64 = C.c_uint64()
        self._inflight = False

    def launch(self, work: WorkDescriptor, grid: Optional[int] = None) -> PhaseTiming:
        if self._inflight:
            raise UsageError("previous task not yet joined")
        d = as_work(work).to_c()
        g = grid or self.grid
        _lib.check(self._lib.lk_baseline_launch(self._h, C.byref(d), g, C.byref(self._u64)))
        self._inflight = True
        timing = PhaseTiming(PHASE_LAUNCH, self._u64.value, full_mask(g))
        self.timings.append(timing)
        return timing

    def wait(self) -> PhaseTiming:
        if not self._inflight:
            raise UsageError("no task in flight")
        _lib.check(self._lib.lk_baseline_wait(self._h, C.byref(self._u64)))
        self._inflight = False
        timing = PhaseTiming(PHASE_WAIT, self._u64.value, full_mask(self.grid))
        self.timings.append(timing)
        return timing

    def bench(self, work: WorkDescriptor, rounds: int, grid: Optional[int] = None):
        d = as_work(work).to_c()
        launch = np.zeros(rounds, dtype=np.uint64)
        total = np.zeros(rounds, dtype=np.uint64)
        _lib.check(self._lib.lk_baseline_bench(self._h, C.byref(d), grid or self.grid, rounds,
                                               launch.ctypes.data, total.ctypes.data))
        return launch, total

    def time_kernel(self, work: WorkDescriptor, reps: int, grid: Optional[int] = None) -> float:
        """Average device ms per launch (CUDA events on the launching stream)."""
        d = work.to_c()
        ms = C.c_float()
        _lib.check(self._lib.lk_baseline_time_kernel(self._h, C.byref(d), grid or self.grid, reps,
                                                     C.byref(ms)))
        return float(ms.value)

    def close(self) -> None:
        if self._h:
            self._lib.lk_baseline_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# The reference's spawn-per-task baseline name, for drop-in call sites.
ThreadSpawnBaseline = LaunchSyncBaseline


def profile_run(cfg: Optional[NativeConfig] = None, rounds: int = 20000, works=()) -> int:
    """Boot, run `rounds` handshakes from a host thread started before the
    kernel launch, and tear down (lk_profile_run): the persistent kernel
    under ncu (--replay-mode application).  No `works`: round-robin empty
    tasks; else full-mask dispatches of works[r % len(works)] (payload
    WorkDescriptors).  Returns the rounds' host wall time in ns."""
    cfg = cfg or NativeConfig(num_workers=None)
    ds = [as_work(w).to_c() for w in works]
    arr = (_lib.lk_desc * max(1, len(ds)))(*ds)
    ns = C.c_uint64()
    _lib.check(_lib.load().lk_profile_run(C.byref(cfg.to_c()), C.cast(arr, C.c_void_p) if ds else None, len(ds),
                                          rounds, C.byref(ns)))
    return ns.value


def sm_topology(device: int = 0) -> list[int]:
    """GPC group of every SM (index = %smid), from clustered probe launches
    (lk_sm_topology).  Call with no session live.  Combine with a session's
    ``smid_map`` to place a latency partition on one GPC, or spread it."""
    n = C.c_int()
    _lib.check(_lib.load().lk_sm_count(device, C.byref(n)))
    out = (C.c_int32 * n.value)()
    groups = C.c_uint32()
    _lib.check(_lib.load().lk_sm_topology(device, out, n.value, C.byref(groups)))
    return list(out)


def workers_by_gpc(smid_map: list[int], topology: list[int]) -> dict[int, list[int]]:
    """{gpc: [worker ids]} for a session's workers."""
    out: dict[int, list[int]] = {}
    for w, sm in enumerate(smid_map):
        out.setdefault(topology[sm] if 0 <= sm < len(topology) else -1, []).append(w)
    return out


def clock_offset(device: int = 0, rounds: int = 2000) -> tuple[int, int]:
    """(globaltimer - CLOCK_MONOTONIC ns, best echo round trip ns)."""
    off, rtt = C.c_int64(), C.c_uint64()
    _lib.check(_lib.load().lk_clock_offset(device, rounds, C.byref(off), C.byref(rtt)))
    return off.value, rtt.value


FLOOR_MODES = {"kernel_sync": _lib.FLOOR_SYNC, "kernel_query": _lib.FLOOR_QUERY, "graph_sync": _lib.FLOOR_GRAPH}


def launch_floor(device: int, mode: str, rounds: int, spin_sched: bool = False):
    """The cheapest conventional launch+sync per task (lk_launch_floor_bench):
    an empty <<<1,32,0>>> kernel joined by stream sync ("kernel_sync"), by a
    host spin on cudaStreamQuery ("kernel_query"), or as a one-node CUDA graph
    ("graph_sync"); spin_sched sets cudaDeviceScheduleSpin (process-wide).
    Returns (total_ns, launch_ns) arrays.  Run with no session live."""
    total = np.zeros(rounds, dtype=np.uint64)
    launch = np.zeros(rounds, dtype=np.uint64)
    _lib.check(_lib.load().lk_launch_floor_bench(device, FLOOR_MODES[mode], 1 if spin_sched else 0, rounds,
                                                 total.ctypes.data, launch.ctypes.data))
    return total, launch


def pingpong(device: int, rounds: int) -> np.ndarray:
    """Raw host->GPU->host word round trips (ns): the link floor under LK."""
    out = np.zeros(rounds, dtype=np.uint64)
    _lib.check(_lib.load().lk_pingpong(device, rounds, out.ctypes.data))
    return out
