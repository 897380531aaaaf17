# SPDX-License-Identifier: Apache-2.0
"""Schedule trace in the reference's JSONL format, and the reference's
bounded-staleness audit over it.

The GPU runtime records the same schedule events as the reference's
ShadowScheduler (dispatch / job_start / job_done / install /
barrier_wait_begin / barrier_wait_end; asg_get_events). This module writes
them exactly as proj/src/trace.cpp:54-115 does (one object per line, keys in
the reference's order, canonical (step, worker, seq) order, integer
microseconds), parses such files (trace.cpp:117-145), and restates
audit_staleness (proj/src/metrics.cpp:131-210), so a GPU run can be audited
with the reference's own rule set and file format.
"""
import json
import math

from . import abi

EVENT_NAMES = {abi.EV_DISPATCH: "dispatch", abi.EV_JOB_START: "job_start", abi.EV_JOB_DONE: "job_done",
               abi.EV_INSTALL: "install", abi.EV_BARRIER_WAIT_BEGIN: "barrier_wait_begin",
               abi.EV_BARRIER_WAIT_END: "barrier_wait_end", abi.EV_PREFETCH: "prefetch", abi.EV_DRAIN: "drain"}


def block_id(spec, param_names=None):
    """BlockSpec::id (precond.cpp:64-67): param[r0:r1,c0:c1]."""
    name = param_names[spec.param_index] if param_names else f"param{spec.param_index}"
    return f"{name}[{spec.row_begin}:{spec.row_end},{spec.col_begin}:{spec.col_end}]"


def events_from_optimizer(opt, worker=0, param_names=None):
    """(step, worker, event, block_id, version, t_micros, seq) rows of an
    AsteriaOptimizer's schedule events, in emission order."""
    ids = {}
    rows = []
    for seq, e in enumerate(opt.events()):
        if e.block not in ids:
            ids[e.block] = block_id(opt.block_info(e.block).spec, param_names)
        rows.append({"step": int(e.step), "worker": int(worker), "event": EVENT_NAMES[e.kind],
                     "block_id": ids[e.block], "version": int(e.version), "t_micros": int(math.floor(e.t_us + 0.5)), "seq": seq})
    return rows


def write_trace(path, per_worker_events):
    """write_trace_file (trace.cpp:86-115) without coherence rows: events
    merged in canonical (step, worker, seq) order, one JSON object per line."""
    allev = [e for evs in per_worker_events for e in evs]
    allev.sort(key=lambda e: (e["step"], e["worker"], e["seq"]))
    with open(path, "w") as f:
        for e in allev:
            f.write('{"step":%d,"worker":%d,"event":"%s","block_id":"%s","version":%d,"t_micros":%d}\n'
                    % (e["step"], e["worker"], e["event"], e["block_id"], e["version"], e["t_micros"]))


def parse_trace(path):
    """parse_trace_file (trace.cpp:117-145): runtime events in file order."""
    out = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line:
                continue
            d = json.loads(line)
            if "event" in d:
                out.append(d)
    return out


def audit_staleness(events, staleness_S, pf, steps):
    """audit_staleness (metrics.cpp:131-210): replays the trace, checks that
    every consumed preconditioner is at most (S+1)*pf steps older than the
    step consuming it and that no block has two jobs in flight (coalescing).
    Returns {assertions, violations, coalescing_violations, max_consumed_age}."""
    audit = {"assertions": 0, "violations": 0, "coalescing_violations": 0, "max_consumed_age": 0}
    blocks = {}
    in_barrier = {}
    bound = (staleness_S + 1) * pf
    current = events[0]["step"] if events else 0

    def state(bid):
        return blocks.setdefault(bid, {"dispatch_steps": [], "pending": 0, "installed": -1, "next": -1})

    def consume_all(step):
        for st in blocks.values():
            if st["installed"] < 0:
                continue
            audit["assertions"] += 1
            age = step - st["installed"]
            audit["max_consumed_age"] = max(audit["max_consumed_age"], age)
            if age > bound:
                audit["violations"] += 1
        for st in blocks.values():  # StepEnd installs become visible next step
            if st["next"] >= 0:
                st["installed"], st["next"] = st["next"], -1

    for e in events:
        if e["step"] != current:
            for s in range(current, e["step"]):
                consume_all(s)
            current = e["step"]
        st = state(e["block_id"] or "-")
        kind = e["event"]
        if kind == "dispatch":
            st["pending"] += 1
            st["dispatch_steps"].append(e["step"])
            audit["assertions"] += 1
            if st["pending"] > 1:
                audit["coalescing_violations"] += 1
        elif kind == "install":
            snap = st["dispatch_steps"].pop(0) if st["dispatch_steps"] else e["step"]
            st["pending"] = max(0, st["pending"] - 1)
            if in_barrier.get(e["worker"], False):
                st["installed"] = snap
            else:
                st["next"] = snap
        elif kind == "barrier_wait_begin":
            in_barrier[e["worker"]] = True
        elif kind == "barrier_wait_end":
            in_barrier[e["worker"]] = False
    if events:
        consume_all(current)
        for s in range(current + 1, steps):
            consume_all(s)
    return audit
