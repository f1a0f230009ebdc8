"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports persistkern from /root/reference/pkg/src (read-only) and records:
  protocol_golden.json   encode/decode results, the worker_step outcome for
                         every (phase, word) pair of interest, complete_work,
                         replay verdicts (first bad index, reason, dispatch
                         counts) for hand-written, randomly generated and
                         corrupted traces, and criterion-7 style sim traces.
  native_golden.json     traces recorded by the reference's own threaded
                         NativeSession for fixed programs, with their
                         per-worker projections.
The fixtures are what the oracle (oracle/) and the B200 runtime are checked
against on machines without the reference.
"""
from __future__ import annotations

import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from persistkern import native, protocol as p  # noqa: E402
from persistkern.calibration import Calibration  # noqa: E402
from persistkern.device import DeviceConfig, WorkDescriptor, build_device  # noqa: E402
from persistkern.errors import ProtocolViolation  # noqa: E402
from persistkern.host import mask_of  # noqa: E402
from persistkern.link import LinkModel, POLICY_INDEFINITE, POLICY_NONE  # noqa: E402
from persistkern.sim import JitterModel, run_until_quiescent  # noqa: E402

PHASES = {"booting": p.Phase.BOOTING, "idle": p.Phase.IDLE, "working": p.Phase.WORKING,
          "finished_pending_ack": p.Phase.FINISHED_PENDING_ACK, "exited": p.Phase.EXITED}
WORDS = list(range(0, 32)) + [0xFFFF, p.WORD_MAX - 1, p.WORD_MAX]


def step_case(phase: str, slot, word: int):
    st = p.WorkerState(PHASES[phase], slot)
    try:
        r = p.worker_step(st, word)
    except ProtocolViolation:
        return {"violation": True}
    act = r.action
    return {"phase": r.state.phase.value, "slot": r.state.slot, "publish": r.publish,
            "action": None if act is None else ("exit" if isinstance(act, p.ExitLoop) else ["begin", act.slot])}


def verdict(trace):
    v, rs = p.replay_trace(trace)
    return {"bad_index": None if v is None else v.index, "reason": None if v is None else v.reason,
            "counts": {str(k): list(c) for k, c in rs.dispatch_counts().items()}}


def reference_trace(rng: random.Random, sms: int, stages: int):
    """A legal trace walked through the reference's worker_step + host rules."""
    trace, states = [], [p.WorkerState(p.Phase.BOOTING) for _ in range(sms)]
    cells = [[p.NOP, p.NOP] for _ in range(sms)]

    def dev(i, complete=False):
        r = p.complete_work(states[i]) if complete else p.worker_step(states[i], cells[i][0])
        states[i] = r.state
        if r.publish is not None and r.publish != cells[i][1]:
            cells[i][1] = r.publish
            trace.append(("D", i, r.publish))

    for i in range(sms):
        dev(i)
        dev(i)
    for _ in range(stages):
        targets = [i for i in range(sms) if rng.random() < 0.7] or [0]
        slot = rng.randrange(4)
        for i in targets:
            trace.append(("H", i, 16 + slot))
            cells[i][0] = 16 + slot
        for i in targets:
            dev(i)
            dev(i, complete=True)
            trace.append(("H", i, 4))
            cells[i][0] = 4
            dev(i)
    for i in range(sms):
        trace.append(("H", i, 8))
        cells[i][0] = 8
        dev(i)
    return trace


def random_program(rng: random.Random, num_sms: int):
    program, slot = [("init",)], 0
    for _ in range(rng.randint(1, 3)):
        sms = rng.sample(range(num_sms), rng.randint(1, num_sms))
        split = rng.randrange(len(sms)) if len(sms) > 1 and rng.random() < 0.3 else 0
        covered = 0
        for group in [g for g in (sms[:split], sms[split:]) if g]:
            program.append(("trigger", mask_of(group), WorkDescriptor(slot=slot, iterations=rng.randrange(400))))
            slot += 1
            covered |= mask_of(group)
        program.append(("wait", covered))
    program.append(("dispose",))
    return program


def protocol_golden():
    g = {"words": {"INIT": p.INIT, "FINISHED": p.FINISHED, "WORKING": p.WORKING, "NOP": p.NOP,
                   "EXIT": p.EXIT, "WORK_BASE": p.WORK_BASE, "MAX_SLOT": p.MAX_SLOT,
                   "board_bytes_16": p.board_bytes(16)}}
    dec = {}
    for w in WORDS:
        try:
            c = p.decode_to_gpu(w)
            dec[str(w)] = ["work", c.slot] if isinstance(c, p.Work) else [type(c).__name__.lower()]
        except ProtocolViolation:
            dec[str(w)] = None
    g["decode"] = dec
    g["encode_work"] = {str(s): p.encode_to_gpu(p.Work(s)) for s in list(range(256)) + [p.MAX_SLOT]}
    steps = []
    for phase, slots in (("booting", [None]), ("idle", [None]), ("working", [0, 5, p.MAX_SLOT]),
                         ("finished_pending_ack", [0, 5, p.MAX_SLOT]), ("exited", [None])):
        for slot in slots:
            for w in WORDS:
                steps.append({"phase": phase, "slot": slot, "word": w, "out": step_case(phase, slot, w)})
    g["step"] = steps
    comp = []
    for phase, slot in (("booting", None), ("idle", None), ("working", 3), ("finished_pending_ack", 3)):
        try:
            r = p.complete_work(p.WorkerState(PHASES[phase], slot))
            comp.append({"phase": phase, "slot": slot, "out": {"phase": r.state.phase.value,
                                                                "slot": r.state.slot, "publish": r.publish}})
        except ProtocolViolation:
            comp.append({"phase": phase, "slot": slot, "out": {"violation": True}})
    g["complete"] = comp

    traces = []
    ok = [("H", 0, 16), ("D", 0, 2), ("D", 0, 1), ("H", 0, 4), ("D", 0, 4)]
    hand = [ok, [], [("D", 0, 0), ("D", 0, 4)] + ok,
            [("H", 0, 16), ("H", 1, 16), ("D", 1, 2), ("D", 0, 2), ("D", 0, 1), ("D", 1, 1), ("H", 1, 4),
             ("H", 0, 4), ("D", 0, 4), ("D", 1, 4)],
            [("H", 0, 16), ("H", 0, 17)], [("H", 0, 9)], [("H", 0, 16), ("D", 0, 9)], [("D", 0, 2)],
            [("H", 0, 4)], [("H", 0, 16), ("D", 0, 2), ("H", 0, 4)], [("H", 0, 16), ("D", 0, 2), ("D", 0, 4)],
            [("H", 0, 16), ("H", 0, 8)], [("H", 0, 8), ("H", 0, 16)], [("H", 0, 8), ("D", 0, 4)],
            [("D", 0, 0), ("D", 0, 0)], [("H", -1, 16)], [("Q", 0, 16)], [("H", 3, 8), ("D", 3, 1)],
            [("H", 0, 16), ("D", 0, 2), ("D", 0, 1), ("H", 0, 8), ("D", 0, 4)]]
    for t in hand:
        traces.append({"kind": "hand", "trace": t, **verdict(t)})
    rng = random.Random(1234)
    for _ in range(60):
        sms = rng.randint(1, 4)
        t = reference_trace(rng, sms, rng.randint(1, 6))
        traces.append({"kind": "legal", "trace": t, **verdict(t)})
    rng = random.Random(99)
    for _ in range(60):
        t = reference_trace(rng, 2, 3)
        idx = rng.randrange(len(t))
        side, sm, _ = t[idx]
        bad = list(t)
        bad[idx] = (side, sm, rng.choice([3, 5, 9, 13, 15]) if side == "H" else rng.choice([3, 5, 8, 9, 16]))
        traces.append({"kind": "corrupt", "trace": bad, "corrupted_index": idx, **verdict(bad)})
    # criterion-7 style: sim executor traces of random programs
    rng = random.Random(20250808)
    cal = Calibration(init_boot_cycles=50, lk_teardown_cycles=50)
    for _ in range(40):
        num_sms = rng.randint(1, 8)
        device = build_device(DeviceConfig(num_sms=num_sms))
        link = LinkModel(deferral_policy=rng.choice([POLICY_NONE, POLICY_INDEFINITE]))
        jitter = JitterModel(seed=rng.randrange(1 << 30), base_range=rng.choice([0, 64]))
        t = run_until_quiescent(device, link, random_program(rng, num_sms), jitter=jitter, cal=cal,
                                workaround_full_board=True).writes()
        traces.append({"kind": "sim", "trace": [list(x) for x in t], **verdict(t)})
    g["traces"] = [{**x, "trace": [list(r) for r in x["trace"]]} for x in traces]
    return g


def native_golden():
    """Programs run on the reference's own threaded executor."""
    programs = {
        "mixed3": (3, [(0b001, 0, "wait"), (0b110, 1, "wait"), (0b111, 2, "wait"), (0b010, 0, "wait")]),
        "split4": (4, [(0b0011, 0, None), (0b1100, 1, None), ("wait", 0b1111), (0b1111, 5, "wait")]),
        "single1": (1, [(1, 0, "wait"), (1, 0, "wait"), (1, 7, "wait")]),
    }
    out = {}
    for name, (n, prog) in programs.items():
        cfg = native.NativeConfig(num_workers=n, spin_yield_threshold=200, record_trace=True)
        s, _ = native.NativeSession.start(cfg)
        dispatched = []
        for item in prog:
            if item[0] == "wait":
                s.wait(item[1])
                continue
            mask, slot, w = item
            s.trigger(mask, WorkDescriptor(slot=slot, iterations=16))
            dispatched.append([mask, slot])
            if w:
                s.wait(mask)
        s.dispose()
        writes = [(r.side, r.sm_id, r.word) for r in s.recorded_trace()]
        proj = {}
        for side, sm, word in writes:
            proj.setdefault(str(sm), []).append([side, word])
        out[name] = {"num_workers": n, "program": dispatched, "writes": [list(w) for w in writes],
                     "projection": proj, **verdict(writes)}
    return out


if __name__ == "__main__":
    (OUT / "protocol_golden.json").write_text(json.dumps(protocol_golden(), separators=(",", ":")))
    (OUT / "native_golden.json").write_text(json.dumps(native_golden(), indent=1))
    print("wrote", OUT / "protocol_golden.json", OUT / "native_golden.json")
