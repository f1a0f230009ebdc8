"""Work descriptors and device payload buffers.

``WorkDescriptor`` keeps the reference's constructor
(/root/reference/pkg/src/persistkern/device.py:48-66: slot, iterations, kind,
data_in_ref, data_out_ref) and adds the payload kinds the B200 worker
executes.  The reference's only kind is ``busy_loop``; its native worker
ignores ``kind`` and the data refs (native.py:179-181).  Here the kind picks
a device work function and the refs are device buffers:

=================== ============================= ===========================
kind                data_in_ref                   data_out_ref
=================== ============================= ===========================
empty               --                            --
busy_loop           --                            --
vector_add_i32      (a, b) int32                  out int32 (may alias a/b)
saxpy_f32           (x, y) float32                out float32 (y for in-place)
block_reduce_f32    x float32                     partials float64[ceil(n/4096)]
                                                  (one per 4096-element block);
                                                  ``total_ref`` float64[1]
hbm_stream          src (any, 4-B elements)       dst
=================== ============================= ===========================

A buffer is a torch CUDA tensor, a :class:`DeviceBuffer`, a
:class:`HostBuffer` or a pinned torch CPU tensor (mapped pinned host memory,
zero-copy), or a raw address (int) of either kind; the runtime classifies every pointer when it stages the
descriptor and refuses anything else.  ``n`` defaults to the element count of
the first input.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .errors import ConfigError, UnsupportedWorkloadError, UsageError

EMPTY = "empty"
BUSY_LOOP = "busy_loop"
VECTOR_ADD_I32 = "vector_add_i32"
SAXPY_F32 = "saxpy_f32"
BLOCK_REDUCE_F32 = "block_reduce_f32"
HBM_STREAM = "hbm_stream"
KINDS = tuple(_lib.KIND_IDS)
SINGLE_THREAD_KINDS = (EMPTY, BUSY_LOOP)

# algorithmic HBM bytes per element
BYTES_PER_ELEMENT = {VECTOR_ADD_I32: 12, SAXPY_F32: 12, BLOCK_REDUCE_F32: 4, HBM_STREAM: 8}
# (block_reduce_f32 also writes 8 B per 4096 elements of block partials: +0.2%)


REDUCE_BLOCK = 4096   # block_reduce_f32: elements per block partial


def reduce_blocks(n: int) -> int:
    """Block partials a block_reduce_f32 of n elements writes (float64 each)."""
    return -(-int(n) // REDUCE_BLOCK)


class DeviceBuffer:
    """A cudaMalloc'd payload buffer owned by the runtime (no torch needed)."""

    def __init__(self, nbytes: int, device: int = 0):
        lib = _lib.load()
        ptr = C.c_uint64()
        _lib.check(lib.lk_dev_alloc(device, nbytes, C.byref(ptr)))
        self.ptr = ptr.value
        self.nbytes = nbytes
        self.device = device

    @classmethod
    def from_array(cls, arr: np.ndarray, device: int = 0) -> "DeviceBuffer":
        buf = cls(arr.nbytes, device)
        buf.upload(arr)
        return buf

    def upload(self, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr)
        if a.nbytes > self.nbytes:
            raise UsageError("array larger than the device buffer")
        _lib.check(_lib.load().lk_memcpy_h2d(self.ptr, a.ctypes.data, a.nbytes))

    def download(self, dtype, count: Optional[int] = None) -> np.ndarray:
        dt = np.dtype(dtype)
        count = self.nbytes // dt.itemsize if count is None else count
        out = np.empty(count, dtype=dt)
        _lib.check(_lib.load().lk_memcpy_d2h(out.ctypes.data, self.ptr, out.nbytes))
        return out

    def free(self) -> None:
        if self.ptr:
            _lib.load().lk_dev_free(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class _HostView:
    """Array-interface holder for HostBuffer.array(): as the view's base it
    keeps the HostBuffer (and so the pinned allocation) referenced."""

    def __init__(self, buf: "HostBuffer", nbytes: int):
        self.buf = buf
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (buf.ptr, False),
                                    "version": 3}


class HostBuffer:
    """Mapped pinned host memory (``lk_host_alloc``: cudaHostAlloc Mapped |
    Portable) that the persistent workers read and write over the link:
    a zero-copy payload buffer.  It replaces the reference's Copyin/Copyout
    phases (P/host.py:212-224) for small transfers, where a cudaMemcpy's fixed
    cost dwarfs the bytes (P/link.py:84-122).

    The runtime classifies the pointer when the descriptor is staged
    (LK_DF_HOSTMEM): the worker reads it with sys-scope loads and publishes
    FINISHED with a sys-scope release, so once ``wait`` returns the outputs
    are in ``array()``.  The device address is the host address (UVA).
    Write inputs before ``trigger`` and read outputs after ``wait``: the
    protocol's handshake is the synchronisation."""

    def __init__(self, nbytes: int, device: int = 0):
        lib = _lib.load()
        host = C.c_void_p()
        _lib.check(lib.lk_host_alloc(device, nbytes, C.byref(host)))
        self.ptr = int(host.value)
        self.nbytes = nbytes
        self.device = device

    @classmethod
    def from_array(cls, arr: np.ndarray, device: int = 0) -> "HostBuffer":
        buf = cls(arr.nbytes, device)
        buf.upload(arr)
        return buf

    def array(self, dtype, count: Optional[int] = None) -> np.ndarray:
        """A numpy view of the buffer (no copy).  The view keeps the buffer
        alive; an explicit ``free()`` invalidates it."""
        if not self.ptr:
            raise UsageError("host buffer freed")
        dt = np.dtype(dtype)
        count = self.nbytes // dt.itemsize if count is None else count
        if count * dt.itemsize > self.nbytes:
            raise UsageError("view larger than the host buffer")
        return np.asarray(_HostView(self, count * dt.itemsize)).view(dt)

    def upload(self, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr)
        if a.nbytes > self.nbytes:
            raise UsageError("array larger than the host buffer")
        C.memmove(self.ptr, a.ctypes.data, a.nbytes)

    def download(self, dtype, count: Optional[int] = None) -> np.ndarray:
        return self.array(dtype, count).copy()

    def free(self) -> None:
        if self.ptr:
            _lib.load().lk_host_free(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _addr(ref) -> int:
    if ref is None:
        return 0
    if isinstance(ref, int):
        return ref
    if isinstance(ref, (DeviceBuffer, HostBuffer)):
        return ref.ptr
    if hasattr(ref, "data_ptr"):
        if hasattr(ref, "is_cuda") and not ref.is_cuda:
            # a pinned CPU tensor is mapped host memory under UVA: zero-copy,
            # like a HostBuffer (the runtime checks the mapping at staging)
            if not (hasattr(ref, "is_pinned") and ref.is_pinned()):
                raise UsageError("payload tensors must live on the GPU or in pinned host memory")
        return int(ref.data_ptr())
    cai = getattr(ref, "__cuda_array_interface__", None)
    if cai is not None:
        return int(cai["data"][0])
    raise UsageError(f"cannot take a device address of {type(ref).__name__}")


def _numel(ref) -> Optional[int]:
    if isinstance(ref, (DeviceBuffer, HostBuffer)):
        return ref.nbytes // 4
    if hasattr(ref, "numel"):
        return int(ref.numel())
    return None


def _nbytes(ref) -> Optional[int]:
    """Size of a payload buffer in bytes, or None for a raw address."""
    if isinstance(ref, (DeviceBuffer, HostBuffer)):
        return ref.nbytes
    if hasattr(ref, "numel") and hasattr(ref, "element_size"):
        return int(ref.numel()) * int(ref.element_size())
    nb = getattr(ref, "nbytes", None)
    if isinstance(nb, int):
        return nb
    cai = getattr(ref, "__cuda_array_interface__", None)
    if cai is not None:
        n = 1
        for d in cai["shape"]:
            n *= int(d)
        return n * np.dtype(cai["typestr"]).itemsize
    return None


def _dtype_name(ref) -> Optional[str]:
    dt = getattr(ref, "dtype", None)
    return None if dt is None else str(dt).replace("torch.", "")


@dataclass(frozen=True)
class WorkDescriptor:
    """One offloadable unit: what the worker runs when ``16+slot`` lands."""

    slot: int
    iterations: int = 0
    kind: str = BUSY_LOOP
    data_in_ref: Optional[object] = field(default=None, compare=False)
    data_out_ref: Optional[object] = field(default=None, compare=False)
    alpha: float = 1.0
    n: Optional[int] = None
    total_ref: Optional[object] = field(default=None, compare=False)

    def __post_init__(self) -> None:
        if self.slot < 0:
            raise ConfigError(f"slot must be nonnegative, got {self.slot}")
        if self.iterations < 0:
            raise ConfigError(f"iterations must be nonnegative, got {self.iterations}")
        if self.kind not in _lib.KIND_IDS:
            raise UnsupportedWorkloadError(f"unknown workload kind {self.kind!r}")
        if self.kind in SINGLE_THREAD_KINDS and (self.data_in_ref is not None
                                                 or self.data_out_ref is not None):
            raise ConfigError(f"{self.kind} work must not carry data references")
        if self.kind not in SINGLE_THREAD_KINDS and (self.data_in_ref is None
                                                     or self.data_out_ref is None):
            raise ConfigError(f"{self.kind} work needs data_in_ref and data_out_ref")

    @property
    def multi_worker(self) -> bool:
        """True when the masked workers shard a payload (the trigger mask matters)."""
        return self.kind not in SINGLE_THREAD_KINDS

    def inputs(self) -> tuple:
        ins = self.data_in_ref
        return tuple(ins) if isinstance(ins, (tuple, list)) else (ins,)

    def elements(self) -> int:
        if self.n is not None:
            return int(self.n)
        if not self.multi_worker:
            return 0
        counts = [c for c in (_numel(r) for r in self.inputs()) if c is not None]
        if not counts:
            raise ConfigError(f"{self.kind}: pass n= for raw device addresses")
        return min(counts)

    def payload_bytes(self) -> int:
        return BYTES_PER_ELEMENT.get(self.kind, 0) * self.elements() * max(1, self.iterations
                                                                           if self.kind == HBM_STREAM else 1)

    def to_c(self) -> "_lib.lk_desc":
        d = _lib.lk_desc()
        d.kind = _lib.KIND_IDS[self.kind]
        d.iterations = self.iterations
        d.alpha = float(self.alpha)
        if not self.multi_worker:
            return d
        ins = self.inputs()
        want = {VECTOR_ADD_I32: ("int32", 2), SAXPY_F32: ("float32", 2),
                BLOCK_REDUCE_F32: ("float32", 1), HBM_STREAM: (None, 1)}[self.kind]
        if len(ins) != want[1]:
            raise ConfigError(f"{self.kind} takes {want[1]} input buffer(s), got {len(ins)}")
        for r in ins + (self.data_out_ref,):
            dn = _dtype_name(r)
            if want[0] and dn is not None and dn != want[0]:
                raise ConfigError(f"{self.kind} expects {want[0]} buffers, got {dn}")
        d.n = self.elements()
        # the kernel writes out[0, n) (maps) and reads in*[0, n): a short
        # buffer would be overrun on the device, so refuse it here
        for r in ins + ((self.data_out_ref,) if self.kind != BLOCK_REDUCE_F32 else ()):
            nb = _nbytes(r)
            if nb is not None and nb < 4 * d.n:
                raise ConfigError(f"{self.kind}: a {nb}-byte buffer cannot hold n={d.n} elements")
        if self.kind == BLOCK_REDUCE_F32:
            nb = _nbytes(self.total_ref)
            if self.total_ref is not None and nb is not None and nb < 8:
                raise ConfigError("block_reduce_f32: total_ref must hold one float64")
            need = 8 * reduce_blocks(d.n)
            nb = _nbytes(self.data_out_ref)
            if nb is not None and nb < need:
                raise ConfigError(f"block_reduce_f32: data_out_ref needs {need} bytes "
                                  f"(one float64 per {REDUCE_BLOCK}-element block), got {nb}")
        d.in0 = _addr(ins[0])
        d.in1 = _addr(ins[1]) if len(ins) > 1 else 0
        d.out = _addr(self.data_out_ref)
        if self.kind == BLOCK_REDUCE_F32:
            d.aux = _addr(self.total_ref)
        if any(p % 16 for p in (d.in0, d.in1, d.out)):
            d.flags |= _lib.DF_SCALAR
        return d


_FOREIGN: dict = {}


def as_work(work) -> WorkDescriptor:
    """Accept the reference's own ``persistkern.device.WorkDescriptor`` (or any
    object with its fields: slot, iterations, kind, data_in_ref, data_out_ref;
    P/device.py:48-66) so existing call sites pass their descriptors unchanged.
    The converted descriptor is cached per source object, so re-triggering the
    same foreign descriptor stays a words-only dispatch."""
    if isinstance(work, WorkDescriptor):
        return work
    hit = _FOREIGN.get(id(work))
    if hit is not None and hit[0] is work:
        return hit[1]
    try:
        conv = WorkDescriptor(slot=work.slot, iterations=getattr(work, "iterations", 0),
                              kind=getattr(work, "kind", BUSY_LOOP),
                              data_in_ref=getattr(work, "data_in_ref", None),
                              data_out_ref=getattr(work, "data_out_ref", None),
                              alpha=getattr(work, "alpha", 1.0), n=getattr(work, "n", None),
                              total_ref=getattr(work, "total_ref", None))
    except AttributeError as exc:
        raise UsageError(f"not a work descriptor: {type(work).__name__}") from exc
    if len(_FOREIGN) > 4096:
        _FOREIGN.clear()
    _FOREIGN[id(work)] = (work, conv)
    return conv
