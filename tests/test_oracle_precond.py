# SPDX-License-Identifier: Apache-2.0
"""Pins the oracle's precond restatement against the reference's own
known-answer tests (proj/tests/precond_test.cpp)."""
import numpy as np
import pytest

import orc
from paper_2605_16184_b200 import abi


def shampoo_cfg():  # precond_test.cpp:20-24
    cfg = orc.defaults_for(abi.SHAMPOO)
    cfg.damping = 0.0
    return cfg


def test_defaults_for():  # precond.cpp:44-62
    a = orc.defaults_for(abi.ADAMW)
    assert a.beta2 == 0.999 and a.accumulation == abi.SUM
    s = orc.defaults_for(abi.SHAMPOO)
    assert s.beta2 == 0.95 and s.accumulation == abi.SUM
    p = orc.defaults_for(abi.SOAP)
    assert p.beta2 == 0.95 and p.accumulation == abi.EMA
    for c in (a, s, p):
        assert (c.lr, c.beta1, c.eps, c.weight_decay, c.precondition_frequency, c.damping,
                c.block_dim_limit) == (1e-3, 0.9, 1e-8, 0.0, 10, 1e-8, 2048)


@pytest.mark.parametrize("field,value", [("precondition_frequency", 0), ("beta1", 1.0), ("beta2", -0.1),
                                         ("lr", -1.0), ("eps", 0.0), ("damping", -1.0),
                                         ("weight_decay", -1.0), ("block_dim_limit", 0)])
def test_validate_rejects(field, value):  # precond.cpp:34-42
    c = orc.defaults_for(abi.SOAP)
    setattr(c, field, value)
    with pytest.raises(abi.ConfigInvalidError):
        orc.validate(c)


def test_accumulate_sum_and_ema():  # precond_test.cpp:72-88
    cfg = shampoo_cfg()
    b = orc.Block(2, 2, abi.SHAMPOO)
    orc.accumulate_factors(b, np.eye(2), cfg)
    assert np.abs(b.factor_l - np.eye(2)).max() == 0.0
    ema = cfg.copy()
    ema.accumulation = abi.EMA
    ema.beta2 = 0.9
    be = orc.Block(2, 2, abi.SHAMPOO)
    orc.accumulate_factors(be, np.sqrt(10.0) * np.eye(2), ema)
    assert be.factor_l[0, 0] == pytest.approx(1.0, rel=1e-12)
    assert be.factor_l[1, 1] == pytest.approx(1.0, rel=1e-12)


def test_accumulate_equals_brute_force():  # precond_test.cpp:90-105
    cfg = shampoo_cfg()
    b = orc.Block(3, 5, abi.SHAMPOO)
    el, er = np.zeros((3, 3)), np.zeros((5, 5))
    for s in range(3):
        g = orc.random_matrix(3, 5, 50 + s)
        orc.accumulate_factors(b, g, cfg)
        gl, gr = g @ g.T, g.T @ g
        el += (gl + gl.T) / 2
        er += (gr + gr.T) / 2
    assert np.abs(b.factor_l - el).max() < 1e-13  # reference: == 0 with Eigen's order
    assert np.abs(b.factor_r - er).max() < 1e-13


def test_refresh_identity_and_scalar_root():  # precond_test.cpp:107-121
    cfg = shampoo_cfg()
    b = orc.Block(2, 2, abi.SHAMPOO)
    b.set(abi.FACTOR_L, np.eye(2))
    b.set(abi.FACTOR_R, np.eye(2))
    r = b.clone()
    orc.refresh_inverse(r, cfg, 7)
    assert r.version == 1 and r.last_refresh_step == 7
    assert np.abs(r.inv_l - np.eye(2)).max() < 1e-14
    b.set(abi.FACTOR_L, 16.0 * np.eye(2))
    r2 = b.clone()
    orc.refresh_inverse(r2, cfg, 8)
    assert np.abs(r2.inv_l - 0.5 * np.eye(2)).max() < 1e-12
    assert np.abs(r2.inv_r - np.eye(2)).max() < 1e-14


def test_refresh_versions_monotonic_and_pure():  # precond_test.cpp:123-137
    cfg = shampoo_cfg()
    cfg.damping = 1e-8
    b = orc.Block(4, 4, abi.SHAMPOO)
    orc.accumulate_factors(b, orc.random_matrix(4, 4, 11), cfg)
    before = b.factor_l
    orc.refresh_inverse(b, cfg, 3)
    assert np.abs(b.factor_l - before).max() == 0.0
    assert b.version == 1
    orc.refresh_inverse(b, cfg, 13)
    assert b.version == 2 and b.last_refresh_step == 13


def test_soap_refresh_under_permutation():  # precond_test.cpp:139-164
    cfg = orc.defaults_for(abi.SOAP)
    b = orc.Block(3, 3, abi.SOAP)
    l = np.diag([1.0, 2.0, 3.0])
    b.set(abi.FACTOR_L, l)
    b.set(abi.FACTOR_R, np.eye(3))
    orc.refresh_inverse(b, cfg, 0)
    v_before = np.abs(orc.random_matrix(3, 3, 21))
    b.set(abi.ROTATED_V, v_before)
    p = np.zeros((3, 3))
    p[0, 2] = p[2, 0] = p[1, 1] = 1.0
    b.set(abi.FACTOR_L, p @ l @ p.T)
    refreshed = b.clone()
    orc.refresh_inverse(refreshed, cfg, 1)
    rot = refreshed.basis_l.T @ b.basis_l
    assert np.abs(np.abs(rot).sum(axis=1) - 1.0).max() < 1e-12
    expect_v = (rot * rot) @ v_before
    assert np.abs(refreshed.rotated_v - expect_v).max() < 1e-12
    assert refreshed.rotated_v.min() >= 0.0


def test_precondition_shampoo_identity_diagonal_oracle():  # precond_test.cpp:166-191
    cfg = shampoo_cfg()
    g = np.diag([2.0, 4.0])
    b = orc.Block(2, 2, abi.SHAMPOO)
    b.set_counters(1)
    assert np.abs(orc.precondition_shampoo(b, g) - g).max() == 0.0
    b2 = orc.Block(2, 2, abi.SHAMPOO)
    orc.accumulate_factors(b2, g, cfg)
    orc.refresh_inverse(b2, cfg, 0)
    t = orc.precondition_shampoo(b2, g)
    assert t[0, 0] == pytest.approx(1.0, rel=1e-10) and t[1, 1] == pytest.approx(1.0, rel=1e-10)
    b3 = orc.Block(8, 8, abi.SHAMPOO)
    g8 = orc.random_matrix(8, 8, 77)
    orc.accumulate_factors(b3, g8, cfg)
    orc.refresh_inverse(b3, cfg, 0)
    il = orc.inv_root_xp(b3.factor_l, 4, 0.0)
    ir = orc.inv_root_xp(b3.factor_r, 4, 0.0)
    assert np.abs(orc.precondition_shampoo(b3, g8) - il @ g8 @ ir).max() < 1e-8


def test_precondition_errors_when_uninitialized():  # precond_test.cpp:193-199
    with pytest.raises(abi.StaleUninitializedError):
        orc.precondition_shampoo(orc.Block(2, 2, abi.SHAMPOO), np.zeros((2, 2)))
    with pytest.raises(abi.StaleUninitializedError):
        orc.precondition_soap(orc.Block(2, 2, abi.SOAP), np.zeros((2, 2)), orc.defaults_for(abi.SOAP))


@pytest.mark.parametrize("c", [0.25, 1.0, 9.0])
def test_shampoo_scalar_factor_invariant(c):  # precond_test.cpp:201-212
    cfg = shampoo_cfg()
    b = orc.Block(5, 3, abi.SHAMPOO)
    b.set(abi.FACTOR_L, c * np.eye(5))
    b.set(abi.FACTOR_R, c * np.eye(3))
    orc.refresh_inverse(b, cfg, 0)
    g = orc.random_matrix(5, 3, 31)
    assert np.abs(orc.precondition_shampoo(b, g) - c ** -0.5 * g).max() < 1e-10


def test_soap_first_step_sign_like():  # precond_test.cpp:214-224
    cfg = orc.defaults_for(abi.SOAP)
    cfg.beta1 = 0.0
    b = orc.Block(2, 3, abi.SOAP)
    b.set_counters(1)
    g = orc.random_matrix(2, 3, 13) * 10.0
    t = orc.precondition_soap(b, g, cfg)
    assert np.allclose(t, np.sign(g), rtol=1e-6, atol=0)


def test_soap_zero_gradient_decays_v():  # precond_test.cpp:226-234
    cfg = orc.defaults_for(abi.SOAP)
    b = orc.Block(2, 2, abi.SOAP)
    b.set_counters(1)
    b.set(abi.ROTATED_V, np.ones((2, 2)))
    t = orc.precondition_soap(b, np.zeros((2, 2)), cfg)
    assert np.abs(t).max() == 0.0
    assert np.abs(b.rotated_v - cfg.beta2).max() < 1e-15


def test_soap_reduces_to_adam_under_identity():  # precond_test.cpp:236-247
    cfg = orc.defaults_for(abi.SOAP)
    b = orc.Block(4, 6, abi.SOAP)
    b.set_counters(1)
    adam = orc.AdamState(4, 6)
    for s in range(20):
        g = orc.random_matrix(4, 6, 400 + s)
        assert np.abs(orc.precondition_soap(b, g, cfg) - orc.adamw_step(adam, g, cfg)).max() < 1e-10


def test_soap_rotation_invariance():  # precond_test.cpp:249-281
    cfg = orc.defaults_for(abi.SOAP)
    n = 4
    u = orc.sym_eig(orc.random_spd(n, 61))[1]
    v = orc.sym_eig(orc.random_spd(n, 62))[1]
    a, bb = orc.Block(n, n, abi.SOAP), orc.Block(n, n, abi.SOAP)
    grads = [orc.random_matrix(n, n, 70 + s) for s in range(4)]
    for g in grads:
        orc.accumulate_factors(a, g, cfg)
        orc.accumulate_factors(bb, u @ g @ v.T, cfg)
    orc.refresh_inverse(a, cfg, 0)
    orc.refresh_inverse(bb, cfg, 0)
    for g in grads:
        ua = orc.precondition_soap(a, g, cfg)
        ub = orc.precondition_soap(bb, u @ g @ v.T, cfg)
        assert np.abs(ub - u @ ua @ v.T).max() < 1e-9
    for s in range(6):
        orc.accumulate_factors(a, orc.random_matrix(n, n, 90 + s), cfg)
        orc.refresh_inverse(a, cfg, s)
        orc.precondition_soap(a, orc.random_matrix(n, n, 80 + s), cfg)
        assert a.rotated_v.min() >= 0.0


def test_adamw_zero_gradient_and_decoupled_decay():  # precond_test.cpp:283-293
    cfg = orc.defaults_for(abi.ADAMW)
    cfg.lr, cfg.weight_decay = 0.1, 0.01
    st = orc.AdamState(2, 2)
    upd = orc.adamw_step(st, np.zeros((2, 2)), cfg)
    assert np.abs(upd).max() == 0.0
    theta = orc.apply_update(np.ones((2, 2)), upd, cfg)
    assert np.abs(theta - (1.0 - cfg.lr * cfg.weight_decay)).max() < 1e-15


def test_adamw_constant_gradient_unit_direction():  # precond_test.cpp:295-303
    cfg = orc.defaults_for(abi.ADAMW)
    st = orc.AdamState(1, 1)
    for _ in range(800):
        u = orc.adamw_step(st, np.array([[0.37]]), cfg)
    assert u[0, 0] == pytest.approx(1.0, rel=1e-4)


def test_adamw_elementwise_loop():  # precond_test.cpp:305-322
    cfg = orc.defaults_for(abi.ADAMW)
    st = orc.AdamState(2, 3)
    m, v = np.zeros(6), np.zeros(6)
    for s in range(1, 51):
        g = orc.random_matrix(2, 3, 600 + s)
        u = orc.adamw_step(st, g, cfg).ravel()
        gk = g.ravel()
        m = cfg.beta1 * m + (1 - cfg.beta1) * gk
        v = cfg.beta2 * v + (1 - cfg.beta2) * gk * gk
        expect = (m / (1 - cfg.beta1 ** s)) / (np.sqrt(v / (1 - cfg.beta2 ** s)) + cfg.eps)
        assert np.allclose(u, expect, rtol=1e-12, atol=0)


def test_apply_update_elementwise():  # precond_test.cpp:324-342
    cfg = orc.defaults_for(abi.ADAMW)
    cfg.lr = 0.0
    theta = orc.random_matrix(3, 3, 91)
    assert np.abs(orc.apply_update(theta, orc.random_matrix(3, 3, 92), cfg) - theta).max() == 0.0
    cfg.lr, cfg.weight_decay = 0.05, 0.2
    upd = orc.random_matrix(3, 3, 93)
    expect = theta - cfg.lr * (upd + cfg.weight_decay * theta)
    assert np.abs(orc.apply_update(theta, upd, cfg) - expect).max() < 1e-15


def make_quadratic(rows, cols, cond, seed):  # precond_test.cpp:358-371
    qa = orc.sym_eig(orc.random_spd(rows, seed))[1]
    qb = orc.sym_eig(orc.random_spd(cols, seed + 1))[1]
    lo = cond ** -0.25
    sa = np.array([lo if i < rows // 2 else 1.0 for i in range(rows)])
    sb = np.array([lo if i < cols // 2 else 1.0 for i in range(cols)])
    a = qa @ np.diag(sa) @ qa.T
    b = qb @ np.diag(sb) @ qb.T
    w_star = 0.3 * orc.random_matrix(rows, cols, seed + 2)
    return a, b, a @ w_star @ b


def steps_to_target(q, method, lr, target, cap):  # precond_test.cpp:373-398
    a, b, c = q
    cfg = orc.defaults_for(method)
    cfg.lr = lr
    cfg.precondition_frequency = 1
    if method == abi.SHAMPOO:
        cfg.accumulation = abi.EMA
    w = np.zeros((a.shape[0], b.shape[1]))
    blk = orc.Block(w.shape[0], w.shape[1], method)
    adam = orc.AdamState(*w.shape)
    for s in range(cap):
        if 0.5 * ((a @ w @ b - c) ** 2).sum() <= target:
            return s
        g = a.T @ (a @ w @ b - c) @ b.T
        if method == abi.ADAMW:
            upd = orc.adamw_step(adam, g, cfg)
        else:
            orc.accumulate_factors(blk, g, cfg)
            orc.refresh_inverse(blk, cfg, s)
            upd = orc.precondition_shampoo(blk, g) if method == abi.SHAMPOO else orc.precondition_soap(blk, g, cfg)
        w = orc.apply_update(w, upd, cfg)
    return cap


def test_shampoo_and_soap_beat_adamw():  # precond_test.cpp:408-419
    q = make_quadratic(8, 6, 1e4, 2024)
    cap, target = 12000, 1e-6

    def best(m):
        return min(steps_to_target(q, m, lr, target, cap) for lr in (1e-3, 3e-3, 1e-2))
    adamw, shampoo, soap = best(abi.ADAMW), best(abi.SHAMPOO), best(abi.SOAP)
    assert shampoo < adamw and soap < adamw
    assert shampoo < cap and soap < cap


def test_replicated_state_roundtrip():  # precond_test.cpp:421-429 (layout precond.cpp:253-265)
    b = orc.Block(3, 2, abi.SHAMPOO)
    b.set(abi.INV_L, 2.0 * np.eye(3))
    flat = orc.replicated_state(b)
    assert flat.size == 9 + 4
    assert np.array_equal(flat[:9].reshape(3, 3), 2.0 * np.eye(3))
    assert np.array_equal(flat[9:].reshape(2, 2), np.eye(2))


# ---- KL-Shampoo (no reference code; properties of our definition) -----------
def test_kl_cold_start_statistics_and_identity_inverses():
    cfg = orc.defaults_for(abi.KL_SHAMPOO)
    b = orc.Block(4, 6, abi.KL_SHAMPOO)
    g = orc.random_matrix(4, 6, 5)
    orc.accumulate_factors(b, g, cfg)
    # Identity start; before any install the inverses are identity:
    # L = b I + (1-b)/n G G^T.
    assert np.abs(b.factor_l - (cfg.beta2 * np.eye(4) + (1 - cfg.beta2) / 6 * g @ g.T)).max() < 1e-14
    assert np.abs(b.factor_r - (cfg.beta2 * np.eye(6) + (1 - cfg.beta2) / 4 * g.T @ g)).max() < 1e-14
    # Cold start passes the gradient through (harness.cpp:458-461 rule).
    assert np.array_equal(orc.step_update(b, g, cfg), g)


def test_kl_refresh_roots_and_inverses():
    cfg = orc.defaults_for(abi.KL_SHAMPOO)
    b = orc.Block(5, 7, abi.KL_SHAMPOO)
    for s in range(12):
        orc.accumulate_factors(b, orc.random_matrix(5, 7, 40 + s), cfg)
    orc.refresh_inverse(b, cfg, 11)
    fl = b.factor_l
    eps = cfg.damping * np.trace(fl) / 5
    d = fl + eps * np.eye(5)
    assert np.abs(b.inv_l @ b.inv_l @ d - np.eye(5)).max() < 1e-9
    assert np.abs(b.get(abi.KL_INV_L) @ d - np.eye(5)).max() < 1e-9
    g = orc.random_matrix(5, 7, 99)
    assert np.abs(orc.precondition_shampoo(b, g) - b.inv_l @ g @ b.inv_r).max() < 1e-14
    # The next statistics use the installed inverses.
    before_l = b.factor_l
    orc.accumulate_factors(b, g, cfg)
    expect = cfg.beta2 * before_l + (1 - cfg.beta2) / 7 * (g @ b.get(abi.KL_INV_R) @ g.T)
    assert np.abs(b.factor_l - (expect + expect.T) / 2).max() < 1e-12


def test_kl_converges_on_quadratic():
    q = make_quadratic(8, 6, 1e4, 2024)
    a, bm, c = q
    cfg = orc.defaults_for(abi.KL_SHAMPOO)
    cfg.lr = 3e-3
    cfg.precondition_frequency = 1
    w = np.zeros((8, 6))
    blk = orc.Block(8, 6, abi.KL_SHAMPOO)
    loss0 = 0.5 * ((a @ w @ bm - c) ** 2).sum()
    for s in range(3000):
        g = a.T @ (a @ w @ bm - c) @ bm.T
        orc.accumulate_factors(blk, g, cfg)
        orc.refresh_inverse(blk, cfg, s)
        w = orc.apply_update(w, orc.precondition_shampoo(blk, g), cfg)
    assert 0.5 * ((a @ w @ bm - c) ** 2).sum() < 1e-3 * loss0
