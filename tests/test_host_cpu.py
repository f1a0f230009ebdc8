"""CPU tests of the boundary and host logic (no GPU): the C-ABI library loads
and exports every symbol include/lk.h declares, struct layouts match the
header, host helpers behave like persistkern.host, foreign descriptors are
accepted, and the scenario-backend aggregation matches the reference's."""
from __future__ import annotations

import ctypes as C
import re
import statistics
from pathlib import Path

import pytest

from paper_2310_01212_b200 import _lib, backend, errors, host, protocol
from paper_2310_01212_b200.device import WorkDescriptor, as_work

ROOT = Path(__file__).resolve().parents[1]
HEADER = (ROOT / "include" / "lk.h").read_text()


def declared_functions() -> set[str]:
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    return set(re.findall(r"\b(lk_[a-z0-9_]+)\s*\(", body))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 35
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) == names   # the binding covers exactly the header


def test_abi_version_and_strerror_without_gpu():
    lib = _lib.load()
    assert lib.lk_abi_version() == 1
    for code in range(0, -11, -1):
        assert lib.lk_strerror(code)
    assert lib.lk_strerror(-99) == b"unknown error"


def test_struct_sizes_match_header():
    assert C.sizeof(_lib.lk_desc) == 64
    assert C.sizeof(_lib.lk_config) == 88
    assert C.sizeof(_lib.lk_trace_rec) == 32
    fields = [f for f, _ in _lib.lk_config._fields_]
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    m = re.search(r"typedef struct lk_config \{(.*?)\} lk_config;", body, re.S)
    hdr = re.findall(r"\b([a-z_]+);", m.group(1))
    assert fields == hdr


def test_error_codes_map_to_reference_exceptions():
    cases = {_lib.LK_E_USAGE: errors.UsageError, _lib.LK_E_BUSY: errors.BusyTriggerError,
             _lib.LK_E_DISPOSE_BUSY: errors.DisposeWhileBusyError, _lib.LK_E_HANG: errors.HangDetected,
             _lib.LK_E_INIT: errors.InitError, _lib.LK_E_CONFIG: errors.ConfigError,
             _lib.LK_E_PROTOCOL: errors.ProtocolViolation}
    for rc, exc in cases.items():
        with pytest.raises(exc):
            _lib.raise_for(rc)
    _lib.check(0)


def test_no_gpu_create_fails_loudly():
    """Without a GPU the product refuses to run: no CPU fallback path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = _lib.lk_config(num_workers=4)
    h, ns = C.c_void_p(), C.c_uint64()
    rc = _lib.load().lk_create(C.byref(cfg), C.byref(h), C.byref(ns))
    assert rc != 0 and not h.value


def test_mask_helpers_match_reference_semantics():
    assert host.full_mask(148) == (1 << 148) - 1
    assert host.sms_in_mask(0b1011) == [0, 1, 3]
    assert host.mask_of([0, 1, 3]) == 0b1011
    with pytest.raises(errors.UsageError):
        host._check_mask(0, 4)
    with pytest.raises(errors.UsageError):
        host._check_mask(1 << 4, 4)
    assert host._check_mask((1 << 148) - 1, 148) == list(range(148))
    assert _lib.mask_bytes(1 << 130, 3) == (1 << 130).to_bytes(24, "little")


def test_phase_timing_contract():
    with pytest.raises(ValueError):
        host.PhaseTiming(host.PHASE_TRIGGER, 5, 0)
    with pytest.raises(ValueError):
        host.PhaseTiming(host.PHASE_INIT, -1)
    csv = host.timings_csv([(0, host.MODEL_LK, host.PhaseTiming(host.PHASE_WAIT, 7, 1))], backend="b200")
    assert csv.splitlines() == ["run_id,model,phase,sm_mask,cycles,backend", "0,LK,Wait,1,7,b200"]


def test_descriptor_validation():
    with pytest.raises(errors.ConfigError):
        WorkDescriptor(slot=-1)
    with pytest.raises(errors.UnsupportedWorkloadError):
        WorkDescriptor(slot=0, kind="matmul")
    with pytest.raises(errors.ConfigError):
        WorkDescriptor(slot=0, kind="busy_loop", data_in_ref=1)
    with pytest.raises(errors.ConfigError):
        WorkDescriptor(slot=0, kind="saxpy_f32")
    d = WorkDescriptor(slot=3, kind="saxpy_f32", data_in_ref=(4096, 8192), data_out_ref=8192,
                       alpha=2.0, n=1000).to_c()
    assert (d.kind, d.n, d.in0, d.in1, d.out, d.flags) == (3, 1000, 4096, 8192, 8192, 0)
    d = WorkDescriptor(slot=3, kind="vector_add_i32", data_in_ref=(4100, 8192), data_out_ref=16,
                       n=7).to_c()
    assert d.flags & _lib.DF_SCALAR


def test_foreign_descriptor_accepted():
    class RefWork:   # shape of persistkern.device.WorkDescriptor (P/device.py:48-66)
        def __init__(self, slot, iterations):
            self.slot, self.iterations, self.kind = slot, iterations, "busy_loop"
            self.data_in_ref = self.data_out_ref = None
    r = RefWork(5, 20_000)
    w = as_work(r)
    assert (w.slot, w.iterations, w.kind) == (5, 20_000, "busy_loop")
    assert as_work(r) is w   # cached: re-triggers stay words-only
    with pytest.raises(errors.UsageError):
        as_work(object())


def test_reference_descriptor_accepted(reference):
    from persistkern.device import WorkDescriptor as RefWork
    w = as_work(RefWork(slot=2, iterations=64))
    assert w.to_c().iterations == 64 and w.to_c().kind == _lib.KIND_IDS["busy_loop"]


def test_backend_aggregate_matches_reference_formula():
    s = [5, 9, 1, 7]
    r = backend.aggregate("LK", "Trigger", s)
    assert (r.avg, r.worst, r.best, r.samples) == (statistics.fmean(s), 9, 1, 4)
    assert r.stddev == statistics.pstdev(s)
    assert backend.aggregate("LK", "Init", [3]).stddev == 0.0
    csv = backend.rows_csv([r])
    assert csv.splitlines()[1].startswith("LK,Trigger,5.5000,9,1,")


def test_backend_aggregate_agrees_with_reference(reference):
    from persistkern import bench as ref_bench
    s = [11, 3, 8]
    mine = backend.aggregate("BASE", "Launch", s)
    theirs = ref_bench._aggregate("BASE", "Launch", s)
    assert (mine.avg, mine.worst, mine.best, mine.stddev, mine.samples) == \
        (theirs.avg, theirs.worst, theirs.best, theirs.stddev, theirs.samples)


def test_trace_file_roundtrip():
    recs = [protocol.TraceRecord(0, "D", 0, protocol.INIT), protocol.TraceRecord(1, "D", 0, protocol.NOP),
            protocol.TraceRecord(2, "H", 0, 16), protocol.TraceRecord(3, "D", 0, protocol.WORKING)]
    text = protocol.format_trace(recs)
    assert protocol.parse_trace(text) == recs
    assert protocol.validate_trace([(r.side, r.sm_id, r.word) for r in recs]) is None


def test_trace_files_validate_with_reference_cli(reference, tmp_path):
    """Trace files written by this runtime's format_trace are accepted by the
    reference's own `persistkern validate` (P/cli.py:223-235), and a corrupted
    one is rejected with exit 1 -- the integration path for device traces."""
    import json
    from persistkern import cli as ref_cli
    golden = json.loads((ROOT / "tests" / "golden" / "native_golden.json").read_text())
    for name, case in golden.items():
        recs = [protocol.TraceRecord(k, s, w, word) for k, (s, w, word) in enumerate(case["writes"])]
        f = tmp_path / f"{name}.trace"
        f.write_text(protocol.format_trace(recs))
        assert ref_cli.main(["validate", str(f)]) == 0, name
        bad = list(recs)
        k = next(i for i, r in enumerate(bad) if r.side == "D" and r.word == protocol.WORKING)
        bad[k] = protocol.TraceRecord(bad[k].step, "D", bad[k].sm_id, protocol.FINISHED)
        g = tmp_path / f"{name}.bad.trace"
        g.write_text(protocol.format_trace(bad))
        assert ref_cli.main(["validate", str(g)]) == 1, name


def test_fast_phase_timing_equals_validated_one():
    from paper_2310_01212_b200 import native
    t = native._timing(host.PHASE_WAIT, 123, 0b101)
    assert t == host.PhaseTiming(host.PHASE_WAIT, 123, 0b101)
    assert hash(t) == hash(host.PhaseTiming(host.PHASE_WAIT, 123, 0b101))
    assert repr(t) == repr(host.PhaseTiming(host.PHASE_WAIT, 123, 0b101))


def test_workers_by_gpc_groups_workers():
    from paper_2310_01212_b200 import native
    topo = [0, 0, 1, 1, 2]
    assert native.workers_by_gpc([4, 0, 3, 1], topo) == {2: [0], 0: [1, 3], 1: [2]}
    assert native.workers_by_gpc([9], topo) == {-1: [0]}


def test_raw_handle_exports_hot_calls():
    raw = _lib.raw()
    assert raw.lk_trigger and raw.lk_wait
    # argtype-free calls on a null session fail cleanly, not crash
    assert raw.lk_wait(None, b"\x01" + b"\x00" * 7, 1, None) == _lib.LK_E_USAGE


def _gpu_trace_program(n):
    """The dispatch program tools/record_gpu_trace.py ran on the B200."""
    full = (1 << n) - 1
    return [(full, 1) if k % 100 == 99 else (1 << (k % n), 0) for k in range(1500)]


def _gpu_trace_records():
    import gzip
    text = gzip.decompress((ROOT / "tests" / "golden" / "gpu_trace_r01.txt.gz").read_bytes()).decode()
    return text, protocol.parse_trace(text)


def test_recorded_b200_trace_replays_clean():
    """A device trace recorded on a B200 (148 workers, 1500 dispatches, with
    full-mask saxpy payloads; tools/record_gpu_trace.py) replays clean in the
    oracle and the native validator, and every worker's projection is the one
    the handshake fixes for the program that ran."""
    from oracle import projection
    from oracle import protocol as O
    _, recs = _gpu_trace_records()
    writes = [(r.side, r.sm_id, r.word) for r in recs]
    n = 148
    assert max(r.sm_id for r in recs) == n - 1
    assert O.replay(writes).violation is None
    assert protocol.validate_trace(writes) is None
    per = projection.program_slots(_gpu_trace_program(n), n)
    proj = projection.projections(writes, n)
    for i in range(n):
        assert proj[i] == projection.expected_projection(per[i]), i


def test_recorded_b200_trace_validates_with_reference_cli(reference, tmp_path):
    """The same B200 trace file passes the reference's own `persistkern
    validate` (P/cli.py:223-235) -- device trace capture feeding the
    reference's validator."""
    from persistkern import cli as ref_cli
    text, _ = _gpu_trace_records()
    f = tmp_path / "b200.trace"
    f.write_text(text)
    assert ref_cli.main(["validate", str(f)]) == 0


def test_timing_log_is_a_list_of_phase_timings():
    import gc
    log = host.TimingLog()
    a = host.PhaseTiming(host.PHASE_TRIGGER, 5, 0b11)
    b = host.PhaseTiming(host.PHASE_WAIT, 9, 0b11)
    log.append(a)
    log.extend([b])
    assert len(log) == 2 and log == [a, b] and list(log) == [a, b]
    assert log[0] == a and log[-1] == b and log[:1] == [a] and a in log
    assert [t.cycles for t in log if t.phase == host.PHASE_WAIT] == [9]
    assert isinstance(log[1], host.PhaseTiming) and hash(log[1]) == hash(b)
    assert list(reversed(log)) == [b, a] and repr(log) == repr([a, b])
    assert log.pop() == b and log == [a]
    log.clear()
    assert not log and log == []
    # rows are untracked by the collector once it has seen them
    log.append(a)
    gc.collect()
    assert not gc.is_tracked(log._rows[0])


_FAKE_LK = r"""
#include <stdint.h>
uint64_t last[4]; uint32_t last_slot, calls;
int fake_trigger(void* h, const uint64_t* m, uint32_t nw, uint32_t slot, const void* d, uint64_t* ns) {
  for (uint32_t k = 0; k < nw && k < 4; ++k) last[k] = m[k];
  last_slot = slot; ++calls; *ns = 1000 + slot;
  return (uintptr_t)h == 7 ? -4 : 0;
}
int fake_wait(void* h, const uint64_t* m, uint32_t nw, uint64_t* ns) {
  for (uint32_t k = 0; k < nw && k < 4; ++k) last[k] = m[k];
  ++calls; *ns = 77;
  return (uintptr_t)h == 7 ? -4 : 0;
}
"""


def _fake_session(tmp_path, handle=1):
    """A NativeSession shell whose C entry points are fakes (no GPU): drives
    the CPython fast path (csrc/lk_pyfast.c) and the Python path side by side."""
    import ctypes as C
    import shutil
    import subprocess
    from paper_2310_01212_b200 import native
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    src = tmp_path / "fake.c"
    src.write_text(_FAKE_LK)
    so = tmp_path / "libfake.so"
    subprocess.run(["gcc", "-O1", "-shared", "-fPIC", str(src), "-o", str(so)], check=True)
    lib = C.CDLL(str(so))
    raw = type("Raw", (), {"lk_trigger": lib.fake_trigger, "lk_wait": lib.fake_wait})
    s = native.NativeSession.__new__(native.NativeSession)
    s.cfg = native.NativeConfig()
    s._lib, s._raw = None, raw
    s._raw_trigger, s._raw_wait = lib.fake_trigger, lib.fake_wait
    s._h, s.num_workers, s.nwords, s.disposed = C.c_void_p(handle), 148, 3, False
    s._fast = None
    s.timings = host.TimingLog()
    s.descriptors, s._staged, s._mask_cache = {}, {}, {}
    s._u64 = C.c_uint64()
    s._u64_ref = C.byref(s._u64)
    s._fast = native._make_fast(s, raw)
    assert s._fast is not None, "_lkfast extension not built"
    return s, lib


def test_pyfast_path_matches_python_path(tmp_path):
    """The C path serves staged descriptors with cached masks; everything it
    declines goes to the Python path (same results, same errors), and the
    session's trigger/wait are the C methods themselves."""
    s, lib = _fake_session(tmp_path)
    calls = C.c_uint32.in_dll(lib, "calls")
    w = WorkDescriptor(slot=3, kind="empty")
    s._staged[3] = (w, 0, False)
    m = (1 << 130) | 1
    # first use: mask not cached -> declined to the Python path (which caches it)
    t1 = s._fast.trigger(m, w)
    assert t1 == host.PhaseTiming(host.PHASE_TRIGGER, 1003, m) and calls.value == 1 and m in s._mask_cache
    assert s._fast.trigger(m, w) == host.PhaseTiming(host.PHASE_TRIGGER, 1003, m)   # now served in C
    assert list((C.c_uint64 * 4).in_dll(lib, "last"))[:3] == [1, 0, 1 << 2]
    assert s._fast.wait(m) == host.PhaseTiming(host.PHASE_WAIT, 77, m)
    assert s.timings == [t1, t1, host.PhaseTiming(host.PHASE_WAIT, 77, m)]
    assert isinstance(s.timings[-1], host.PhaseTiming)
    # declined cases take the Python path: restaging, foreign objects, bad masks
    w2 = WorkDescriptor(slot=3, kind="empty")          # equal fields, different object
    assert s._fast.trigger(m, w2).cycles == 1003 and s._staged[3][0] is w2
    with pytest.raises(errors.UsageError):
        s._fast.trigger(m, object())                   # not a work descriptor
    s._mask_cache[0] = bytes(24)
    s._mask_cache[1 << 148] = bytes(24)
    with pytest.raises(errors.UsageError):
        s._fast.wait(0)                                # the reference's empty-mask error
    with pytest.raises(errors.UsageError):
        s._fast.wait(1 << 148)                         # wider than the workers
    pay = WorkDescriptor(slot=4, kind="empty")
    s._staged[4] = (pay, m, True)                      # staged for mask m only
    n = calls.value
    s._mask(1)
    s._fast.trigger(1, pay)                            # another worker set: restaged by the Python path
    assert calls.value == n + 1 and s._staged[4] == (pay, 0, False)
    # the bound methods: a session's trigger/wait are the C ones
    s._bind_fast()
    assert s.trigger.__self__ is s._fast and s.wait.__self__ is s._fast
    assert s.trigger(m, w2).phase == host.PHASE_TRIGGER
    s._unbind_fast()
    assert "trigger" not in s.__dict__ and s.trigger.__func__ is type(s).trigger
    # rebinding timings keeps both paths appending to the new log
    s._bind_fast()
    s.timings = []
    s.wait(m)
    assert len(s.timings) == 1 and s.timings[0].phase == host.PHASE_WAIT


def test_pyfast_error_codes_raise(tmp_path):
    from paper_2310_01212_b200.errors import HangDetected
    s, _ = _fake_session(tmp_path, handle=7)          # fakes return LK_E_HANG (-4)
    w = WorkDescriptor(slot=0, kind="empty")
    s._staged[0] = (w, 0, False)
    s._mask(1)
    with pytest.raises(HangDetected):
        s._fast.trigger(1, w)                         # C path, raised through _raise_lk
    s._bind_fast()
    with pytest.raises(HangDetected):
        s.trigger(1, w)
    with pytest.raises(HangDetected) as ei:
        s.wait(1)
    assert ei.value.sm_ids == (0,)
    assert len(s.timings) == 0


def test_ack_delay_config():
    from paper_2310_01212_b200 import native
    c = native.NativeConfig().to_c()
    assert c.ack_delay_ns == 300 and not c.flags & (_lib.CF_NO_ACK_DELAY | _lib.CF_ACK_FIXED)
    assert native.NativeConfig(ack_adaptive=False).to_c().flags & _lib.CF_ACK_FIXED
    assert c.idle_delay_ns == 0
    c = native.NativeConfig(ack_delay_ns=0, idle_delay_ns=300).to_c()
    assert c.flags & _lib.CF_NO_ACK_DELAY and c.idle_delay_ns == 300
    for bad in (-1, 100_001):
        with pytest.raises(errors.UsageError):
            native.NativeConfig(ack_delay_ns=bad)


def test_profile_run_refuses_non_direct_configs():
    from paper_2310_01212_b200 import native
    for cfg in (native.NativeConfig(poll_mode="gateway"), native.NativeConfig(record_trace=True)):
        with pytest.raises(errors.ConfigError):
            native.profile_run(cfg, 10)


def test_illegal_word_injection_into_a_b200_trace_is_detected():
    """Criterion 7's injection check (T/test_acceptance.py:168-176,
    T/test_protocol.py:277-291) on the device trace recorded on a B200: an
    illegal word at a random position is caught by the oracle replay and by
    the product validator, at or before that position."""
    import random
    from oracle import protocol as O
    _, recs = _gpu_trace_records()
    writes = [(r.side, r.sm_id, r.word) for r in recs]
    rng = random.Random(20250808)
    for _ in range(60):
        idx = rng.randrange(len(writes))
        side, sm, _ = writes[idx]
        bad = list(writes)
        bad[idx] = (side, sm, rng.choice([3, 5, 9, 13, 15]))
        v = O.replay(bad).violation          # (index, reason)
        assert v is not None and v[0] <= idx
        pv = protocol.validate_trace(bad)
        assert pv is not None and pv.index <= idx


def test_committed_bench_line_keeps_the_contract():
    """The bench line committed under profiles/ carries every key the driver
    and the judge read (bench contract), with the roofline and baseline
    objects complete."""
    import json
    d = json.loads((ROOT / "profiles" / "r01_bench_line.json").read_text())
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "clocks",
              "gpu_launches"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["n_gpus"] >= 1 and d["value"] > 0 and "workload" in d["config"]
    assert set(d["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
    assert set(d["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert abs(d["roofline"]["frac"] - d["roofline"]["achieved"] / d["roofline"]["peak"]) < 1e-3
    assert set(d["cpu_baseline"]) >= {"value", "unit", "cores", "kind", "sample"}
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["gpu_launches"] >= 1
    r = json.loads((ROOT / "profiles" / "r01_bench_reference_line.json").read_text())
    assert r["impl"] == "reference" and r["metric"] == d["metric"] and r["unit"] == d["unit"]
    assert set(r["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}


def test_timing_log_mutable_sequence_surface_matches_list():
    """Every list operation a caller of the reference's ``timings: list``
    (P/native.py:99) could use gives what the same operation on a list gives."""
    import collections.abc as abc
    ts = [host.PhaseTiming(host.PHASE_TRIGGER, k, 0b1) for k in range(1, 6)]
    log, ref = host.TimingLog(ts), list(ts)
    assert isinstance(log, abc.MutableSequence)
    extra = host.PhaseTiming(host.PHASE_WAIT, 99, 0b10)
    for op in (lambda x: x.insert(1, extra), lambda x: x.__setitem__(0, extra),
               lambda x: x.__delitem__(2), lambda x: x.__setitem__(slice(0, 2), [ts[4], ts[3]])):
        op(log)
        op(ref)
        assert log == ref and list(log) == ref
    assert log.index(ts[3]) == ref.index(ts[3]) and log.count(ts[3]) == ref.count(ts[3]) == 2
    assert log.count(extra) == ref.count(extra) == 0
    assert log.copy() == ref and isinstance(log.copy(), list)
