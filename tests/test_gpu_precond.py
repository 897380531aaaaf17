# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the per-block optimizer functions (through the C-ABI) with the
CPU oracle, replaying proj/tests/precond_test.cpp where it applies.

Stated tolerances (fp32 path, 3xTF32 tensor-core products, fp64 refresh):
  * statistics (accumulate_factors):   normwise rel. error <= steps x (1e-6 + 1.2e-8 K)
                                        (K = contraction length; the tensor-core
                                        fp32 accumulation error grows ~linearly in K)
  * refresh (roots / bases / values):  computed from the GPU's own factor,
                                        agree with the fp64 oracle to 1e-6
                                        (fp32 rounding of the stored result)
  * preconditioned update:             normwise rel. error <= 1e-5
where normwise rel. error = max|x - x_ref| / max|x_ref|.
"""
import numpy as np
import pytest

import orc
from paper_2605_16184_b200 import abi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_16184_b200 import precond, runtime
    assert runtime.device_supported(0)
    return precond


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def shampoo_cfg(P):  # precond_test.cpp:20-24
    c = P.defaults_for(abi.SHAMPOO)
    c.damping = 0.0
    return c


def test_accumulate_sum_and_ema_kats(P):  # precond_test.cpp:72-88
    cfg = shampoo_cfg(P)
    b = P.PrecondBlock(2, 2, abi.SHAMPOO, cfg)
    P.accumulate_factors(b, np.eye(2), cfg)
    assert np.abs(b.factor_l - np.eye(2)).max() == 0.0
    ema = cfg.copy()
    ema.accumulation = abi.EMA
    ema.beta2 = 0.9
    be = P.PrecondBlock(2, 2, abi.SHAMPOO, ema)
    P.accumulate_factors(be, np.sqrt(10.0) * np.eye(2), ema)
    assert be.factor_l[0, 0] == pytest.approx(1.0, rel=1e-6)
    assert be.factor_l[1, 1] == pytest.approx(1.0, rel=1e-6)


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.SOAP, abi.KL_SHAMPOO])
@pytest.mark.parametrize("m,n", [(3, 5), (48, 80), (200, 130), (256, 768)])
def test_accumulate_matches_oracle(P, method, m, n):  # precond_test.cpp:90-105 generalised
    cfg = P.defaults_for(method)
    b = P.PrecondBlock(m, n, method, cfg)
    o = orc.Block(m, n, method)
    for s in range(3):
        g = orc.random_matrix(m, n, 50 + s) / np.sqrt(n)
        P.accumulate_factors(b, g, cfg)
        orc.accumulate_factors(o, g, cfg)
    assert rel(b.factor_l, o.factor_l) < 3 * (1e-6 + 1.2e-8 * n)
    assert rel(b.factor_r, o.factor_r) < 3 * (1e-6 + 1.2e-8 * m)
    # exactly symmetric (mirrored epilogue)
    fl = b.factor_l
    assert np.array_equal(fl, fl.T)


def test_refresh_identity_and_scalar_root(P):  # precond_test.cpp:107-121
    cfg = shampoo_cfg(P)
    b = P.PrecondBlock(2, 2, abi.SHAMPOO, cfg)
    b.set(abi.FACTOR_L, np.eye(2))
    b.set(abi.FACTOR_R, np.eye(2))
    P.refresh_inverse(b, cfg, 7)
    assert b.version == 1 and b.last_refresh_step == 7
    assert np.abs(b.inv_l - np.eye(2)).max() < 1e-7
    b.set(abi.FACTOR_L, 16.0 * np.eye(2))
    P.refresh_inverse(b, cfg, 8)
    assert np.abs(b.inv_l - 0.5 * np.eye(2)).max() < 1e-7
    assert np.abs(b.inv_r - np.eye(2)).max() < 1e-7
    assert b.version == 2


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
@pytest.mark.parametrize("m,n", [(8, 8), (33, 64), (130, 96)])
def test_refresh_roots_match_oracle(P, method, m, n):
    cfg = P.defaults_for(method)
    b = P.PrecondBlock(m, n, method, cfg)
    for s in range(4):
        P.accumulate_factors(b, orc.random_matrix(m, n, 70 + s), cfg)
    P.refresh_inverse(b, cfg, 3)
    o = orc.Block(m, n, method)
    o.set(abi.FACTOR_L, b.factor_l)  # identical (fp32-valued) factor
    o.set(abi.FACTOR_R, b.factor_r)
    orc.refresh_inverse(o, cfg, 3)
    assert rel(b.inv_l, o.inv_l) < 1e-6
    assert rel(b.inv_r, o.inv_r) < 1e-6
    if method == abi.KL_SHAMPOO:
        assert rel(b.get(abi.KL_INV_L), o.get(abi.KL_INV_L)) < 1e-6
        assert rel(b.get(abi.KL_INV_R), o.get(abi.KL_INV_R)) < 1e-6


def test_refresh_rejects_indefinite(P):  # densela_test.cpp:110-115 via compute_refresh
    cfg = shampoo_cfg(P)
    b = P.PrecondBlock(2, 2, abi.SHAMPOO, cfg)
    b.set(abi.FACTOR_L, np.diag([1.0, -2.0]))
    b.set(abi.FACTOR_R, np.eye(2))
    with pytest.raises(abi.NotPsdError):
        P.refresh_inverse(b, cfg, 0)
    assert b.version == 0


def test_precondition_shampoo_kats_and_oracle(P):  # precond_test.cpp:166-191
    cfg = shampoo_cfg(P)
    g = np.diag([2.0, 4.0])
    b = P.PrecondBlock(2, 2, abi.SHAMPOO, cfg)
    b.set_counters(1)
    assert np.abs(P.precondition_shampoo(b, g) - g).max() == 0.0
    b2 = P.PrecondBlock(2, 2, abi.SHAMPOO, cfg)
    P.accumulate_factors(b2, g, cfg)
    P.refresh_inverse(b2, cfg, 0)
    t = P.precondition_shampoo(b2, g)
    assert t[0, 0] == pytest.approx(1.0, rel=1e-6) and t[1, 1] == pytest.approx(1.0, rel=1e-6)
    b3 = P.PrecondBlock(8, 8, abi.SHAMPOO, cfg)
    g8 = orc.random_matrix(8, 8, 77)
    P.accumulate_factors(b3, g8, cfg)
    P.refresh_inverse(b3, cfg, 0)
    il = orc.inv_root_xp(b3.factor_l, 4, 0.0)
    ir = orc.inv_root_xp(b3.factor_r, 4, 0.0)
    assert rel(P.precondition_shampoo(b3, g8), il @ g8 @ ir) < 1e-5


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
@pytest.mark.parametrize("m,n", [(64, 96), (256, 384), (768, 256)])
def test_precondition_matches_oracle(P, method, m, n):
    cfg = P.defaults_for(method)
    b = P.PrecondBlock(m, n, method, cfg)
    rng = np.random.default_rng(m + n)
    b.set(abi.INV_L, (lambda a: a @ a.T / m + np.eye(m))(rng.standard_normal((m, m))))
    b.set(abi.INV_R, (lambda a: a @ a.T / n + np.eye(n))(rng.standard_normal((n, n))))
    b.set_counters(1)
    g = rng.standard_normal((m, n))
    out = P.precondition_shampoo(b, g)
    ref = b.inv_l @ g @ b.inv_r  # the installed (fp32-stored) roots, in fp64
    assert rel(out, ref) < 1e-5


def test_precondition_errors_when_uninitialized(P):  # precond_test.cpp:193-199
    b = P.PrecondBlock(2, 2, abi.SHAMPOO)
    with pytest.raises(abi.StaleUninitializedError):
        P.precondition_shampoo(b, np.zeros((2, 2)))
    bs = P.PrecondBlock(2, 2, abi.SOAP)
    with pytest.raises(abi.StaleUninitializedError):
        P.precondition_soap(bs, np.zeros((2, 2)))


@pytest.mark.parametrize("c", [0.25, 1.0, 9.0])
def test_shampoo_scalar_factor_invariant(P, c):  # precond_test.cpp:201-212
    cfg = shampoo_cfg(P)
    b = P.PrecondBlock(5, 3, abi.SHAMPOO, cfg)
    b.set(abi.FACTOR_L, c * np.eye(5))
    b.set(abi.FACTOR_R, c * np.eye(3))
    P.refresh_inverse(b, cfg, 0)
    g = orc.random_matrix(5, 3, 31)
    assert rel(P.precondition_shampoo(b, g), c ** -0.5 * g) < 1e-6


def test_soap_first_step_sign_like(P):  # precond_test.cpp:214-224
    cfg = P.defaults_for(abi.SOAP)
    cfg.beta1 = 0.0
    b = P.PrecondBlock(2, 3, abi.SOAP, cfg)
    b.set_counters(1)
    g = orc.random_matrix(2, 3, 13) * 10.0
    assert np.allclose(P.precondition_soap(b, g, cfg), np.sign(g), rtol=1e-5, atol=0)


def test_soap_zero_gradient_decays_v(P):  # precond_test.cpp:226-234
    cfg = P.defaults_for(abi.SOAP)
    b = P.PrecondBlock(2, 2, abi.SOAP, cfg)
    b.set_counters(1)
    b.set(abi.ROTATED_V, np.ones((2, 2)))
    t = P.precondition_soap(b, np.zeros((2, 2)), cfg)
    assert np.abs(t).max() == 0.0
    assert np.abs(b.rotated_v - cfg.beta2).max() < 1e-7


def test_soap_reduces_to_adam_under_identity(P):  # precond_test.cpp:236-247
    cfg = P.defaults_for(abi.SOAP)
    b = P.PrecondBlock(4, 6, abi.SOAP, cfg)
    b.set_counters(1)
    adam = orc.AdamState(4, 6)
    for s in range(20):
        g = orc.random_matrix(4, 6, 400 + s)
        assert rel(P.precondition_soap(b, g, cfg), orc.adamw_step(adam, g, cfg)) < 1e-5


@pytest.mark.parametrize("m,n", [(4, 6), (40, 24), (128, 200)])
def test_soap_refresh_and_steps_match_oracle(P, m, n):
    """Refreshes happen once the factors are full rank (>= 2 accumulations
    here). In an exactly rank-deficient direction of a factor the rotated
    gradient is pure rounding noise, and Adam's normalisation m/(sqrt(v)+eps)
    turns fp32 noise (~1e-7 |G| > eps = 1e-8) into O(1) update components
    where the fp64 reference's noise (~1e-16 |G|) stays below eps; parity is
    stated for full-rank factors (or |G| * 2^-23 < eps)."""
    cfg = P.defaults_for(abi.SOAP)
    b = P.PrecondBlock(m, n, abi.SOAP, cfg)
    o = orc.Block(m, n, abi.SOAP)
    for s in range(7):
        g = orc.random_matrix(m, n, 900 + s)
        P.accumulate_factors(b, g, cfg)
        orc.accumulate_factors(o, g, cfg)
        if s in (2, 5):
            P.refresh_inverse(b, cfg, s)
            # install the oracle refresh of the GPU's own factor snapshot
            src = orc.Block(m, n, abi.SOAP)
            src.set(abi.FACTOR_L, b.factor_l)
            src.set(abi.FACTOR_R, b.factor_r)
            orc.refresh_from(o, src, cfg, s)
            # eigenvalues agree; bases agree up to column signs
            assert rel(b.get(abi.EIGVALS_L), o.get(abi.EIGVALS_L)) < 1e-10
            ql, qo = b.basis_l, o.basis_l
            assert np.abs(np.abs(np.sum(ql * qo, axis=0)) - 1.0).max() < 1e-8
            # use the GPU's (sign-chosen) bases in the oracle so moments are comparable
            o.set(abi.BASIS_L, ql)
            o.set(abi.BASIS_R, b.basis_r)
            o.set(abi.ROTATED_M, b.rotated_m)
            o.set(abi.ROTATED_V, b.rotated_v)
        # cold-start rule before the first install (harness.cpp:458-461)
        upd = (P.precondition_soap if b.version else P.soap_scaled_step)(b, g, cfg)
        ref = (orc.precondition_soap if o.version else orc.soap_scaled_step)(o, g, cfg)
        assert rel(upd, ref) < 2e-5
        assert b.rotated_v.min() >= 0.0


def test_soap_refresh_under_permutation(P):  # precond_test.cpp:139-164
    cfg = P.defaults_for(abi.SOAP)
    b = P.PrecondBlock(3, 3, abi.SOAP, cfg)
    l = np.diag([1.0, 2.0, 3.0])
    b.set(abi.FACTOR_L, l)
    b.set(abi.FACTOR_R, np.eye(3))
    P.refresh_inverse(b, cfg, 0)
    v_before = np.abs(orc.random_matrix(3, 3, 21))
    b.set(abi.ROTATED_V, v_before)
    q_old = b.basis_l
    p = np.zeros((3, 3))
    p[0, 2] = p[2, 0] = p[1, 1] = 1.0
    b.set(abi.FACTOR_L, p @ l @ p.T)
    P.refresh_inverse(b, cfg, 1)
    rot = b.basis_l.T @ q_old
    assert np.abs(np.abs(rot).sum(axis=1) - 1.0).max() < 1e-12
    assert rel(b.rotated_v, (rot * rot) @ v_before) < 1e-6
    assert b.rotated_v.min() >= 0.0


def test_kl_cold_start_and_statistics(P):
    cfg = P.defaults_for(abi.KL_SHAMPOO)
    b = P.PrecondBlock(40, 72, abi.KL_SHAMPOO, cfg)
    o = orc.Block(40, 72, abi.KL_SHAMPOO)
    for s in range(5):
        g = orc.random_matrix(40, 72, 60 + s)
        P.accumulate_factors(b, g, cfg)
        orc.accumulate_factors(o, g, cfg)
        if s == 2:
            P.refresh_inverse(b, cfg, s)
            src = orc.Block(40, 72, abi.KL_SHAMPOO)
            src.set(abi.FACTOR_L, b.factor_l)
            src.set(abi.FACTOR_R, b.factor_r)
            orc.refresh_from(o, src, cfg, s)
            o.set(abi.FACTOR_L, b.factor_l)
            o.set(abi.FACTOR_R, b.factor_r)
    assert rel(b.factor_l, o.factor_l) < 2e-5
    assert rel(b.factor_r, o.factor_r) < 2e-5


def test_shape_mismatch(P):
    b = P.PrecondBlock(4, 4, abi.SHAMPOO)
    with pytest.raises(abi.ShapeMismatchError):
        P.accumulate_factors(b, np.zeros((3, 4)))
    with pytest.raises(abi.NonFiniteError):
        P.accumulate_factors(b, np.full((4, 4), np.nan))
