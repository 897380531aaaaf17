# SPDX-License-Identifier: Apache-2.0
"""Pins the oracle's bounded-staleness schedule against the reference's own
tests (proj/tests/asyncsched_test.cpp). The Rig below replays the
reference's Rig (asyncsched_test.cpp:13-56) step for step."""
import numpy as np
import pytest

import orc
from paper_2605_16184_b200 import abi


class Rig:  # asyncsched_test.cpp:13-56
    def __init__(self, S, pf, delay_steps, method=abi.SHAMPOO, n=4):
        self.opt = orc.defaults_for(method)
        self.opt.precondition_frequency = pf
        self.cfg = abi.scheduler_defaults()
        self.cfg.staleness_S = S
        self.cfg.pf = pf
        self.cfg.inject_job_delay_steps = delay_steps
        self.cfg.step_compute_us = 1000.0
        self.cfg.install_cost_us = 5.0
        self.sched = orc.Scheduler(self.opt, self.cfg, seed=99)
        self.block = orc.Block(n, n, method)
        self.n = n

    def step(self, s, grad_seed):
        self.sched.advance(self.cfg.step_compute_us)
        orc.accumulate_factors(self.block, orc.random_matrix(self.n, self.n, grad_seed), self.opt)
        self.sched.maybe_dispatch(self.block, 0, s)
        waited = self.sched.staleness_barrier(self.block, 0, s)
        if self.block.version > 0:
            upd = orc.precondition_shampoo(self.block, orc.random_matrix(self.n, self.n, grad_seed + 1))
            assert np.isfinite(upd).all()
        self.sched.step_end([self.block], [0], s)
        return waited

    def count(self, kind, from_step=0):
        return sum(1 for e in self.sched.events() if e.kind == kind and e.step >= from_step)


def test_fresh_stats_zero():  # asyncsched_test.cpp:60-69
    st = Rig(5, 10, 0.0).sched.stats()
    assert (st.dispatched, st.completed, st.installed, st.coalesced, st.wait_total_us, st.pending) == (0, 0, 0, 0, 0.0, 0)


def test_dispatch_only_at_pf_boundaries():  # asyncsched_test.cpp:71-76
    rig = Rig(5, 10, 0.0)
    for s in range(25):
        rig.step(s, 100 + s)
    assert rig.sched.stats().dispatched == 3
    assert rig.count(abi.EV_DISPATCH) == 3


def test_pending_jobs_coalesce():  # asyncsched_test.cpp:78-89
    rig = Rig(100, 10, 25.0)
    for s in range(30):
        rig.step(s, 200 + s)
    st = rig.sched.stats()
    assert st.dispatched == 1 and st.coalesced == 2 and st.pending == 0
    assert rig.block.version == 1


def test_s0_installs_every_boundary():  # asyncsched_test.cpp:91-101
    rig = Rig(0, 10, 2.0)
    for s in range(35):
        w = rig.step(s, 300 + s)
        if s % 10 == 0:
            assert w == pytest.approx(2000.0)
        else:
            assert w == 0.0
    st = rig.sched.stats()
    assert st.dispatched == 4 and st.installed == 4 and rig.block.version == 4


def test_fast_jobs_hide_under_budget():  # asyncsched_test.cpp:103-115
    rig = Rig(3, 10, 2.0)
    total = sum(rig.step(s, 400 + s) for s in range(40))
    assert total == 0.0
    assert rig.count(abi.EV_BARRIER_WAIT_BEGIN) == 0
    rec = rig.sched.freshness(0)
    assert rec.installed_version == rig.block.version
    assert rec.last_install_step == 32


def test_barrier_engages_at_age_s_plus_1():  # asyncsched_test.cpp:117-129
    S = 2
    rig = Rig(S, 10, S + 3.0)
    for s in range(20):
        rig.step(s, 500 + s)
    waits = [e.step for e in rig.sched.events() if e.kind == abi.EV_BARRIER_WAIT_BEGIN]
    assert waits == [S + 1, 10 + S + 1]


def test_counters_conserved():  # asyncsched_test.cpp:131-144
    rig = Rig(1, 5, 1.0)
    last_d = last_i = 0
    for s in range(26):
        rig.step(s, 600 + s)
        st = rig.sched.stats()
        assert st.dispatched >= last_d and st.installed >= last_i
        last_d, last_i = st.dispatched, st.installed
    st = rig.sched.stats()
    assert st.dispatched == st.installed + st.pending


def test_snapshot_isolation():  # asyncsched_test.cpp:146-164
    rig = Rig(100, 10, 3.0)
    rig.sched.advance(1000.0)
    orc.accumulate_factors(rig.block, np.eye(4), rig.opt)
    at_dispatch = rig.block.factor_l
    assert rig.sched.maybe_dispatch(rig.block, 0, 0)
    for k in range(50):
        orc.accumulate_factors(rig.block, orc.random_matrix(4, 4, 700 + k), rig.opt)
    rig.sched.advance(10000.0)
    rig.sched.step_end([rig.block], [0], 5)
    assert rig.block.version == 1
    expect = orc.inv_root(at_dispatch, 4, rig.opt.damping * np.trace(at_dispatch) / 4.0)
    assert np.abs(rig.block.inv_l - expect).max() < 1e-14


def test_installed_inverses_whole_and_finite():  # asyncsched_test.cpp:166-176
    rig = Rig(4, 2, 1.5)
    for s in range(60):
        rig.step(s, 800 + s)
        if rig.block.version > 0:
            m = rig.block.inv_l
            assert np.isfinite(m).all()
            assert np.abs(m - m.T).max() < 1e-12


def test_dispatch_fails_when_pool_down():  # asyncsched_test.cpp:178-184
    rig = Rig(0, 1, 0.0)
    rig.step(0, 900)
    rig.sched.stop_pool()
    orc.accumulate_factors(rig.block, np.eye(4), rig.opt)
    with pytest.raises(abi.WorkerPoolDownError):
        rig.sched.maybe_dispatch(rig.block, 0, 1)


def test_freshness_records():  # asyncsched_test.cpp:186-200
    rig = Rig(10, 10, 4.0)
    rig.step(0, 950)
    rec0 = rig.sched.freshness(0)
    assert rec0.installed_version == 0 and rec0.dispatch_step_of_pending == 0
    for s in range(1, 11):
        rig.step(s, 950 + s)
    rec = rig.sched.freshness(0)
    assert rec.installed_version == 1 and rec.last_install_step == 4
    assert rec.dispatch_step_of_pending == 10 and rec.installed_snapshot_step == 0


def test_consumed_age_bounded_under_coalescing():  # asyncsched_test.cpp:202-217
    rig = Rig(1, 1, 3.0)
    worst = 0
    for s in range(40):
        rig.step(s, 7000 + s)
        if rig.block.version > 0:
            worst = max(worst, s - rig.sched.freshness(0).installed_snapshot_step)
    assert worst <= (1 + 1) * 1


def test_jitter_stream_deterministic():
    """Jitter draws come from mt19937_64 seeded as asyncsched.cpp:248."""
    def run():
        rig = Rig(3, 2, 0.5)
        rig.cfg.inject_job_delay_jitter_steps = 2.0
        rig.sched = orc.Scheduler(rig.opt, rig.cfg, seed=7)
        for s in range(30):
            rig.step(s, 10 + s)
        return [(e.step, e.kind, e.t_us) for e in rig.sched.events()]
    assert run() == run()
