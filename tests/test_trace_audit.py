# SPDX-License-Identifier: Apache-2.0
"""Schedule trace (reference JSONL format, proj/src/trace.cpp:54-145) and the
reference's staleness audit (proj/src/metrics.cpp:131-210) restated in
paper_2605_16184_b200/trace.py; the GPU case audits a real event-mode run."""
import pytest

from paper_2605_16184_b200 import trace as T


def ev(step, event, block="w[0:8,0:8]", worker=0, version=0, t=0, seq=0):
    return {"step": step, "worker": worker, "event": event, "block_id": block, "version": version,
            "t_micros": t, "seq": seq}


def test_trace_format_and_canonical_order(tmp_path):
    w1 = [ev(1, "install", worker=1, seq=0), ev(0, "dispatch", worker=1, seq=1)]
    w0 = [ev(1, "dispatch", worker=0, seq=0, version=3, t=12), ev(0, "install", worker=0, seq=1)]
    p = tmp_path / "trace.jsonl"
    T.write_trace(p, [w1, w0])
    lines = p.read_text().splitlines()
    # canonical (step, worker, seq) order, the reference's key order and spacing (trace.cpp:54-69)
    assert lines[0] == '{"step":0,"worker":0,"event":"install","block_id":"w[0:8,0:8]","version":0,"t_micros":0}'
    assert lines[1].startswith('{"step":0,"worker":1,"event":"dispatch"')
    assert lines[2] == '{"step":1,"worker":0,"event":"dispatch","block_id":"w[0:8,0:8]","version":3,"t_micros":12}'
    back = T.parse_trace(p)
    assert [(e["step"], e["worker"], e["event"]) for e in back] == [(0, 0, "install"), (0, 1, "dispatch"),
                                                                   (1, 0, "dispatch"), (1, 1, "install")]


def test_audit_synchronous_refresh_is_fresh():
    # S = 0, pf = 1: dispatch, barrier-install every step (asyncsched_test.cpp:91-101)
    events = []
    for s in range(5):
        events += [ev(s, "dispatch"), ev(s, "barrier_wait_begin"), ev(s, "install"), ev(s, "barrier_wait_end")]
    a = T.audit_staleness(events, staleness_S=0, pf=1, steps=5)
    assert a["violations"] == 0 and a["coalescing_violations"] == 0
    assert a["max_consumed_age"] == 0
    assert a["assertions"] == 5 + 5  # one dispatch and one consumption per step


def test_audit_step_end_install_visible_next_step():
    # dispatched at 0, installed at StepEnd of step 2 -> consumed from step 3 with age 3
    events = [ev(0, "dispatch"), ev(2, "install")]
    a = T.audit_staleness(events, staleness_S=2, pf=1, steps=5)
    assert a["max_consumed_age"] == 4  # step 4 consumes the step-0 snapshot
    assert a["violations"] == 1        # bound (S+1)*pf = 3 < 4


def test_audit_detects_coalescing_violation():
    events = [ev(0, "dispatch"), ev(1, "dispatch")]
    assert T.audit_staleness(events, 1, 1, 2)["coalescing_violations"] == 1


@pytest.mark.gpu
def test_gpu_event_mode_run_passes_the_reference_audit(tmp_path):
    torch = pytest.importorskip("torch")
    from paper_2605_16184_b200 import abi, runtime
    from paper_2605_16184_b200.optimizer import AsteriaOptimizer
    opt = runtime.optimizer_defaults(abi.SOAP)
    opt.block_dim_limit, opt.precondition_frequency = 128, 3
    sched = runtime.scheduler_defaults()
    sched.pf, sched.staleness_S, sched.install_mode = 3, 2, abi.INSTALL_EVENT
    sched.refresh_mode = abi.REFRESH_F32
    g = torch.Generator(device="cuda").manual_seed(0)
    params = [torch.randn(256, 256, device="cuda", generator=g) * 0.1]
    grads = [torch.zeros_like(params[0])]
    o = AsteriaOptimizer(params, grads, opt, sched)
    steps = 20
    for s in range(steps):
        grads[0].normal_(generator=g).mul_(1e-3)
        o.step(s)
    o.synchronize()
    p = tmp_path / "gpu_trace.jsonl"
    T.write_trace(p, [T.events_from_optimizer(o, param_names=["w"])])
    a = T.audit_staleness(T.parse_trace(p), staleness_S=2, pf=3, steps=steps)
    assert a["violations"] == 0 and a["coalescing_violations"] == 0, a
    assert a["max_consumed_age"] <= (2 + 1) * 3
    assert a["assertions"] > 0
