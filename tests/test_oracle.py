"""CPU tests: pin the oracle to the reference's golden vectors, then check the
product's host-compiled state machine and native trace validator against the
same vectors.  (No GPU needed.)"""
from __future__ import annotations

import json
import random
from pathlib import Path

import numpy as np
import pytest

from oracle import cpu_session, projection
from oracle import protocol as O
from paper_2310_01212_b200 import protocol as L
from paper_2310_01212_b200.errors import ProtocolViolation

GOLDEN = Path(__file__).resolve().parent / "golden"
PG = json.loads((GOLDEN / "protocol_golden.json").read_text())
NG = json.loads((GOLDEN / "native_golden.json").read_text())

PH = {"booting": O.BOOT, "idle": O.IDLE, "working": O.WORK, "finished_pending_ack": O.FIN,
      "exited": O.GONE}
LPH = {"booting": L.Phase.BOOTING, "idle": L.Phase.IDLE, "working": L.Phase.WORKING,
       "finished_pending_ack": L.Phase.FINISHED_PENDING_ACK, "exited": L.Phase.EXITED}


def _oracle_step(case):
    try:
        ph, sl, pub, act = O.step(PH[case["phase"]], case["slot"], case["word"])
    except O.Illegal:
        return {"violation": True}
    if act == "exit":
        a = "exit"
    elif act is None:
        a = None
    else:
        a = ["begin", act[1]]
    return {"phase": ph, "slot": sl, "publish": pub, "action": a}


def _product_step(case):
    try:
        r = L.worker_step(L.WorkerState(LPH[case["phase"]], case["slot"]), case["word"])
    except ProtocolViolation:
        return {"violation": True}
    act = r.action
    a = None if act is None else ("exit" if isinstance(act, L.ExitLoop) else ["begin", act.slot])
    return {"phase": r.state.phase.value, "slot": r.state.slot, "publish": r.publish, "action": a}


# ---------------------------------------------------------------- words

def test_word_values_match_reference():
    w = PG["words"]
    assert (O.INIT, O.FINISHED, O.WORKING, O.NOP, O.EXIT, O.WORK_BASE) == (
        w["INIT"], w["FINISHED"], w["WORKING"], w["NOP"], w["EXIT"], w["WORK_BASE"])
    assert (L.INIT, L.FINISHED, L.WORKING, L.NOP, L.EXIT, L.WORK_BASE, L.MAX_SLOT) == (
        w["INIT"], w["FINISHED"], w["WORKING"], w["NOP"], w["EXIT"], w["WORK_BASE"], w["MAX_SLOT"])
    assert L.board_bytes(16) == w["board_bytes_16"]


def test_decode_golden():
    for word, want in PG["decode"].items():
        word = int(word)
        try:
            c = O.command(word)
            got = [c[0], c[1]] if c[0] == "work" else [c[0]]
        except O.Illegal:
            got = None
        assert got == want, word
        try:
            lc = L.decode_to_gpu(word)
            lgot = ["work", lc.slot] if isinstance(lc, L.Work) else [type(lc).__name__.lower()]
        except ProtocolViolation:
            lgot = None
        assert lgot == want, word


def test_encode_golden():
    for slot, word in PG["encode_work"].items():
        assert L.encode_to_gpu(L.Work(int(slot))) == word
    with pytest.raises(ProtocolViolation):
        L.encode_to_gpu(L.Work(L.MAX_SLOT + 1))
    with pytest.raises(ProtocolViolation):
        L.encode_to_gpu(L.Work(-1))


# ---------------------------------------------------------------- state machine

def test_oracle_step_table_matches_reference():
    assert len(PG["step"]) > 200
    for case in PG["step"]:
        assert _oracle_step(case) == case["out"], case


def test_product_state_machine_matches_reference():
    """The __host__ __device__ lk_worker_step the kernel runs, on every golden case."""
    for case in PG["step"]:
        assert _product_step(case) == case["out"], case


def test_complete_work_golden():
    for case in PG["complete"]:
        want = case["out"]
        try:
            ph, sl, pub, _ = O.complete(PH[case["phase"]], case["slot"])
            got = {"phase": ph, "slot": sl, "publish": pub}
        except O.Illegal:
            got = {"violation": True}
        assert got == want
        try:
            r = L.complete_work(L.WorkerState(LPH[case["phase"]], case["slot"]))
            lgot = {"phase": r.state.phase.value, "slot": r.state.slot, "publish": r.publish}
        except ProtocolViolation:
            lgot = {"violation": True}
        assert lgot == want


# ---------------------------------------------------------------- replay

def _counts(d):
    return {str(k): list(v) for k, v in d.items()}


@pytest.mark.parametrize("kind", ["hand", "legal", "corrupt", "sim"])
def test_oracle_replay_golden(kind):
    cases = [t for t in PG["traces"] if t["kind"] == kind]
    assert cases
    for t in cases:
        trace = [tuple(r) for r in t["trace"]]
        r = O.replay(trace)
        got = None if r.violation is None else r.violation[0]
        assert got == t["bad_index"], t
        if r.violation is not None:
            assert r.violation[1] == t["reason"]
        assert _counts(r.dispatch_counts()) == t["counts"]


@pytest.mark.parametrize("kind", ["hand", "legal", "corrupt", "sim"])
def test_native_validator_golden(kind):
    """csrc/lk_validate.cpp (the product's validator) on the same vectors."""
    for t in (t for t in PG["traces"] if t["kind"] == kind):
        trace = [tuple(r) for r in t["trace"]]
        v, rs = L.replay_trace(trace)
        assert (None if v is None else v.index) == t["bad_index"], t
        if v is not None:
            assert v.reason == t["reason"]
        assert _counts(rs.dispatch_counts()) == t["counts"]


def test_corruptions_detected_at_or_before_index():
    for t in (t for t in PG["traces"] if t["kind"] == "corrupt"):
        assert t["bad_index"] is not None and t["bad_index"] <= t["corrupted_index"]


def test_validator_random_agreement():
    """Oracle and native validator agree on random (mostly illegal) traces."""
    rng = random.Random(7)
    for _ in range(3000):
        n = rng.randint(0, 12)
        trace = [(rng.choice("HD"), rng.randint(0, 2), rng.choice([0, 1, 2, 3, 4, 8, 9, 16, 17, 20]))
                 for _ in range(n)]
        o = O.replay(trace)
        v, rs = L.replay_trace(trace)
        assert (None if o.violation is None else o.violation) == (None if v is None else (v.index, v.reason))
        assert o.dispatch_counts() == rs.dispatch_counts()


# ---------------------------------------------------------------- native-session goldens

def test_native_golden_projection_formula():
    for name, g in NG.items():
        assert g["bad_index"] is None
        per = projection.program_slots([tuple(x) for x in g["program"]], g["num_workers"])
        for w in range(g["num_workers"]):
            got = [tuple(x) for x in g["projection"][str(w)]]
            assert got == projection.expected_projection(per[w]), (name, w)


def test_cpu_port_traces_validate_and_project():
    s = cpu_session.CpuSession(num_workers=3, spin_yield_threshold=200, record_trace=True)
    s.start()
    prog = [(0b001, 0), (0b110, 1), (0b111, 2), (0b010, 0)]
    for mask, slot in prog:
        s.trigger(mask, slot, iterations=16)
        s.wait(mask)
    s.dispose()
    w = s.writes()
    r = O.replay(w)
    assert r.violation is None
    per = projection.program_slots(prog, 3)
    proj = projection.projections(w, 3)
    for i in range(3):
        assert proj[i] == projection.expected_projection(per[i])
    assert all(a == b for a, b in r.dispatch_counts().values())


# ---------------------------------------------------------------- live reference (build box only)

def test_oracle_agrees_with_live_reference(reference):
    rp = reference["protocol"]
    rng = random.Random(11)
    for _ in range(4000):
        n = rng.randint(0, 14)
        trace = [(rng.choice("HD"), rng.randint(0, 2), rng.choice([0, 1, 2, 3, 4, 8, 9, 16, 17, 21]))
                 for _ in range(n)]
        v, rs = rp.replay_trace(trace)
        o = O.replay(trace)
        assert (None if v is None else (v.index, v.reason)) == o.violation
        assert rs.dispatch_counts() == o.dispatch_counts()


def test_cpu_port_matches_live_reference_projection(reference):
    native = reference["native"]
    from persistkern.device import WorkDescriptor
    cfg = native.NativeConfig(num_workers=2, spin_yield_threshold=200, record_trace=True)
    rs, _ = native.NativeSession.start(cfg)
    port = cpu_session.CpuSession(num_workers=2, spin_yield_threshold=200, record_trace=True)
    port.start()
    for k in range(20):
        m = 1 << (k % 2) if k % 3 else 0b11
        rs.trigger(m, WorkDescriptor(slot=k % 3, iterations=8))
        rs.wait(m)
        port.trigger(m, k % 3, 8)
        port.wait(m)
    rs.dispose()
    port.dispose()
    ref_w = [(r.side, r.sm_id, r.word) for r in rs.recorded_trace()]
    assert projection.projections(ref_w, 2) == projection.projections(port.writes(), 2)


# ---------------------------------------------------------------- properties

def test_product_state_machine_walks_match_the_oracle():
    """Property check beyond the goldens (hypothesis): random walks of words
    -- legal ones, gap words, slots up to MAX_SLOT -- through the product's
    __host__ __device__ state machine and through the reference-pinned
    oracle give the same phase, slot, publish and action at every step, and
    a violation at the same step.  A begun item is completed the way the
    worker completes it (complete_work) before the walk goes on."""
    hypothesis = pytest.importorskip("hypothesis")
    st = hypothesis.strategies
    words = st.one_of(st.sampled_from([O.NOP, O.EXIT, 0, 1, 2, 3, 5, 9, 15]),
                      st.integers(O.WORK_BASE, O.WORK_BASE + 40),
                      st.integers(O.WORK_BASE, 0xFFFFFFFF))

    @hypothesis.settings(max_examples=400, deadline=None)
    @hypothesis.given(st.lists(words, min_size=1, max_size=40))
    def walk(seq):
        case = {"phase": O.BOOT, "slot": None}
        for w in seq:
            case["word"] = w
            want, got = _oracle_step(case), _product_step(case)
            assert got == want, (case, got, want)
            if "violation" in want or want["action"] == "exit":
                return
            if want["action"] is not None:   # began work: the worker completes it
                ph, sl, _pub, _ = O.complete(want["phase"], want["slot"])
                case = {"phase": ph, "slot": sl}
            else:
                case = {"phase": want["phase"], "slot": want["slot"]}
    walk()


def _reduce_scalar(x):
    """A literal, loop-by-loop restatement of block_reduce_f32's order of
    operations (lk_kernels.cu: block_sum_smem / block_sum_global /
    reduce_finish) to pin the vectorised oracle on small inputs."""
    n = len(x)
    nb = -(-n // 4096)
    parts = []
    for b in range(nb):
        lanes = []
        for lane in range(32):
            h = [[np.float32(0.0)] * 4, [np.float32(0.0)] * 4]   # even-k and odd-k accumulators
            for k in range(32):
                v = lane + 32 * k
                for c in range(4):
                    e = b * 4096 + 4 * v + c
                    if e < n:
                        h[k & 1][c] = np.float32(h[k & 1][c] + x[e])   # fp32, round to nearest
            a = [float(np.float32(h[0][c] + h[1][c])) for c in range(4)]
            lanes.append((a[0] + a[1]) + (a[2] + a[3]))
        o = 16
        while o >= 1:
            lanes = [lanes[i] + lanes[i ^ o] for i in range(32)]
            o //= 2
        parts.append(lanes[0])
    s = [0.0] * 512
    for i, p in enumerate(parts):
        s[i % 512] = s[i % 512] + p
    o = 256
    while o >= 1:
        s = [s[j] + s[j ^ o] for j in range(512)]
        o //= 2
    return parts, s[0]


@pytest.mark.parametrize("n", [0, 1, 7, 4096, 4101, 9000])
def test_block_reduce_oracle_matches_scalar_restatement(n):
    from oracle import work as W
    x = np.random.default_rng(n).uniform(-1, 1, n).astype(np.float32)
    parts, tot = _reduce_scalar(x)
    np.testing.assert_array_equal(W.block_reduce_partials(x), np.array(parts, dtype=np.float64))
    assert W.block_reduce_total(x) == tot


def test_block_reduce_oracle_exact_on_integers_and_close_on_uniform():
    from oracle import work as W
    x = np.random.default_rng(1).integers(0, 8, 1 << 20).astype(np.float32)
    assert W.block_reduce_total(x) == float(x.astype(np.float64).sum())
    u = np.random.default_rng(2).uniform(0, 1, 1 << 20).astype(np.float32)
    assert abs(W.block_reduce_total(u) - float(u.astype(np.float64).sum())) <= 1e-8 * float(u.sum())   # fp32 lane sums of 32 values: far inside rtol 1e-6
