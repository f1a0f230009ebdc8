"""ctypes binding of liblk.so (include/lk.h).

ctypes.CDLL drops the GIL for the duration of every foreign call, so the
C-side spins in lk_wait / lk_bench_roundtrip never block other Python
threads.  The library is built in-tree by ``paper_2310_01212_b200.build``;
there is no fallback: a missing library is an ImportError-grade failure.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "liblk.so"

LK_OK = 0
LK_E_USAGE = -1
LK_E_BUSY = -2
LK_E_DISPOSE_BUSY = -3
LK_E_HANG = -4
LK_E_INIT = -5
LK_E_WORKER_DIED = -6
LK_E_CUDA = -7
LK_E_CONFIG = -8
LK_E_PROTOCOL = -9
LK_E_TRACE_LOST = -10

KIND_IDS = {
    "empty": 0,
    "busy_loop": 1,
    "vector_add_i32": 2,
    "saxpy_f32": 3,
    "block_reduce_f32": 4,
    "hbm_stream": 5,
}
DF_SCALAR = 1
DF_HOSTMEM = 2
CF_ACQUIRE_POLL = 1
CF_FENCE_ALWAYS = 2
CF_LSU_PAYLOAD = 4
CF_TIMELINE = 8
CF_LAZY_ACK = 16
CF_ACK_WINDOW = 32
CF_DYNAMIC_TILES = 64
CF_NO_ACK_DELAY = 128
CF_ACK_FIXED = 256
CF_HOST_DESC = 512
CF_FULL_BOARD = 1024
CF_RELAXED_POLL = 2048
FLOOR_SYNC = 0
FLOOR_QUERY = 1
FLOOR_GRAPH = 2
POLL_DIRECT = 0
POLL_GATEWAY = 1
POLL_HYBRID = 2
HINT_EMPTY = 1
HINT_SYSMEM = 4

WERR_NAMES = {
    0: "none",
    1: "illegal to_gpu word",
    2: "work slot triggered while busy with another slot",
    3: "work slot triggered before the previous slot was acknowledged",
    4: "worker stepped after exit",
    5: "work slot outside the device descriptor table",
    6: "unsupported work kind",
    7: "completion signalled outside WORKING",
}


class lk_desc(C.Structure):
    _fields_ = [
        ("kind", C.c_uint32),
        ("flags", C.c_uint32),
        ("iterations", C.c_uint64),
        ("n", C.c_uint64),
        ("in0", C.c_uint64),
        ("in1", C.c_uint64),
        ("out", C.c_uint64),
        ("aux", C.c_uint64),
        ("alpha", C.c_float),
        ("reserved", C.c_uint32),
    ]


class lk_config(C.Structure):
    _fields_ = [
        ("num_workers", C.c_uint32),
        ("threads_per_worker", C.c_uint32),
        ("device", C.c_int32),
        ("spin_strategy", C.c_uint32),
        ("spin_yield_threshold", C.c_uint32),
        ("record_trace", C.c_uint32),
        ("trace_capacity", C.c_uint32),
        ("poll_backoff_ns", C.c_uint32),
        ("cell_stride", C.c_uint32),
        ("num_slots", C.c_uint32),
        ("wait_timeout_ns", C.c_uint64),
        ("flags", C.c_uint32),
        ("poll_replicas", C.c_uint32),
        ("poll_spacing_ns", C.c_uint32),
        ("poll_mode", C.c_uint32),
        ("status_stride", C.c_uint32),
        ("ring_stages", C.c_uint32),
        ("sm_partition", C.c_uint32),
        ("ack_delay_ns", C.c_uint32),
        ("idle_delay_ns", C.c_uint32),
        ("tma_min_workers", C.c_uint32),
    ]


class lk_trace_rec(C.Structure):
    _fields_ = [
        ("step", C.c_uint64),
        ("side", C.c_uint32),
        ("worker", C.c_uint32),
        ("word", C.c_uint32),
        ("hseq", C.c_uint32),
        ("t_ns", C.c_uint64),
    ]


assert C.sizeof(lk_desc) == 64
assert C.sizeof(lk_trace_rec) == 32

P = C.c_void_p
U32 = C.c_uint32
U64 = C.c_uint64
I32 = C.c_int
PU32 = C.POINTER(C.c_uint32)
PU64 = C.POINTER(C.c_uint64)
PI64 = C.POINTER(C.c_int64)
MASK = C.c_char_p   # little-endian u64 words packed by int.to_bytes

# name -> (restype, argtypes); every symbol include/lk.h declares
SIGNATURES = {
    "lk_create": (I32, [C.POINTER(lk_config), C.POINTER(P), PU64]),
    "lk_dispose": (I32, [P, PU64]),
    "lk_destroy": (I32, [P]),
    "lk_abort": (I32, [P, U64]),
    "lk_register_desc": (I32, [P, U32, C.POINTER(lk_desc), MASK, U32]),
    "lk_trigger": (I32, [P, MASK, U32, U32, C.POINTER(lk_desc), PU64]),
    "lk_wait": (I32, [P, MASK, U32, PU64]),
    "lk_read_cells": (I32, [P, PU32, PU32, PU32, U32]),
    "lk_worker_error": (I32, [P, U32, PU32, PU32]),
    "lk_debug_poke": (I32, [P, U32, U32]),
    "lk_smid_map": (I32, [P, PU32, U32]),
    "lk_num_workers": (I32, [P, PU32]),
    "lk_pending": (I32, [P, PU64, U32]),
    "lk_kernel_alive": (I32, [P, PU32]),
    "lk_trace_count": (I32, [P, PU64]),
    "lk_trace_read": (I32, [P, C.POINTER(lk_trace_rec), U64, PU64]),
    "lk_protocol_step": (I32, [PU32, PU32, U32, PU32, PU32, PU32]),
    "lk_protocol_complete": (I32, [PU32, PU32, PU32, PU32]),
    "lk_validate_trace": (I32, [P, P, P, U64, PI64, C.c_char_p, U32, PU64, U32, PU32]),
    "lk_bench_roundtrip": (I32, [P, MASK, U32, U32, U32, U64, P, P, P]),
    "lk_bench_roundtrip_gaps": (I32, [P, MASK, U32, U32, U32, U64, P, P, P, P]),
    "lk_profile_run": (I32, [C.POINTER(lk_config), P, U32, U64, C.POINTER(C.c_uint64)]),
    "lk_last_spans": (I32, [P, P, P, U32]),
    "lk_last_timeline": (I32, [P, P, U32]),
    "lk_last_host_times": (I32, [P, P, U32]),
    "lk_fast_count": (I32, [P, P, U32]),
    "lk_launch_floor_bench": (I32, [I32, U32, U32, U64, P, P]),
    "lk_clock_offset": (I32, [I32, U32, PI64, PU64]),
    "lk_sm_topology": (I32, [I32, C.POINTER(C.c_int32), U32, PU32]),
    "lk_pingpong": (I32, [I32, U64, P]),
    "lk_baseline_create": (I32, [I32, U32, C.POINTER(P)]),
    "lk_baseline_launch": (I32, [P, C.POINTER(lk_desc), U32, PU64]),
    "lk_baseline_wait": (I32, [P, PU64]),
    "lk_baseline_bench": (I32, [P, C.POINTER(lk_desc), U32, U64, P, P]),
    "lk_baseline_time_kernel": (I32, [P, C.POINTER(lk_desc), U32, U32, C.POINTER(C.c_float)]),
    "lk_baseline_destroy": (I32, [P]),
    "lk_baseline_set_tma": (I32, [P, I32]),
    "lk_baseline_create_in": (I32, [P, U32, C.POINTER(P)]),
    "lk_partition_info": (I32, [P, PU32, PU32]),
    "lk_pin_thread_near": (I32, [I32, PU32]),
    "lk_device_count": (I32, [C.POINTER(C.c_int)]),
    "lk_sm_count": (I32, [I32, C.POINTER(C.c_int)]),
    "lk_dev_alloc": (I32, [I32, U64, PU64]),
    "lk_dev_free": (I32, [U64]),
    "lk_host_alloc": (I32, [I32, U64, C.POINTER(P)]),
    "lk_host_free": (I32, [P]),
    "lk_memcpy_h2d": (I32, [U64, P, U64]),
    "lk_memcpy_d2h": (I32, [P, U64, U64]),
    "lk_strerror": (C.c_char_p, [I32]),
    "lk_last_error": (C.c_char_p, []),
    "lk_abi_version": (U32, []),
}

_lib = None


def load() -> C.CDLL:
    """Load liblk.so (built on demand); never falls back to anything else."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() or os.environ.get("LK_REBUILD"):
        from .build import build
        build()
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_raw = None


def raw() -> C.CDLL:
    """The same library through a second handle whose functions carry no
    argtypes: for the per-task hot calls (lk_trigger, lk_wait) whose
    arguments the caller already passes as ctypes-ready objects, skipping
    ctypes' per-argument conversion (~40% of the call cost)."""
    global _raw
    if _raw is None:
        load()
        _raw = C.CDLL(str(LIB_PATH))
    return _raw


def last_error() -> str:
    return load().lk_last_error().decode(errors="replace")


def raise_for(rc: int, *, sm_ids=()) -> None:
    """Map an LK_E_* status to the persistkern exception taxonomy."""
    if rc == LK_OK:
        return
    msg = last_error() or load().lk_strerror(rc).decode()
    if rc == LK_E_USAGE:
        raise errors.UsageError(msg)
    if rc == LK_E_BUSY:
        raise errors.BusyTriggerError(msg)
    if rc == LK_E_DISPOSE_BUSY:
        raise errors.DisposeWhileBusyError(msg)
    if rc == LK_E_HANG:
        raise errors.HangDetected(msg, sm_ids=tuple(sm_ids))
    if rc == LK_E_INIT:
        raise errors.InitError(msg)
    if rc == LK_E_WORKER_DIED:
        raise errors.UsageError(msg)
    if rc == LK_E_CONFIG:
        raise errors.ConfigError(msg)
    if rc == LK_E_PROTOCOL:
        raise errors.ProtocolViolation(msg)
    if rc == LK_E_TRACE_LOST:
        raise errors.TraceLostError(msg)
    raise errors.CudaError(msg)


def check(rc: int, **kw) -> None:
    if rc != LK_OK:
        raise_for(rc, **kw)


def mask_bytes(mask: int, nwords: int) -> bytes:
    return mask.to_bytes(8 * nwords, "little")
