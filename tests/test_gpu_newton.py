# SPDX-License-Identifier: Apache-2.0
"""The NEWTON refresh (asg_refresh_mode ASG_REFRESH_NEWTON): Shampoo's
L^-1/4 and KL-Shampoo's L^-1/2 and L^-1 by coupled Newton-Schulz iterations
on the tensor cores (asg_newton.cu), replayed against the oracle's
inv_root (densela.hpp:267-282 via compute_refresh precond.cpp:129-142) on the
refresh cases of tests/test_gpu_refresh_f32.py.

Stated tolerances (normwise relative against the fp64 oracle run on the GPU's
own fp32 factor): roots <= 2e-5 (the F32 rows of DESIGN.md §4); the
iteration stops once max|M - I| <= 1e-3 and takes one more X step, which
leaves ~1e-6 (quadratic convergence), below the fp32 factor's own noise.
Trajectories as tests/test_gpu_step.py with r = 5e-4."""
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


def newton_sched():
    s = abi.scheduler_defaults()
    s.refresh_mode = abi.REFRESH_NEWTON
    return s


PRECS = [pytest.param(abi.PREC_3XTF32, id="3xtf32"), pytest.param(abi.PREC_3XF16, id="3xf16")]


@pytest.mark.parametrize("precision", PRECS)
@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
@pytest.mark.parametrize("m,n", [(8, 8), (33, 64), (130, 96), (256, 200)])
def test_newton_roots_match_oracle(P, method, m, n, precision):
    """3XF16: the iterates as scaled fp16 pairs (asg_newton.cu header); same bound."""
    cfg = P.defaults_for(method)
    b = P.PrecondBlock(m, n, method, cfg, precision=precision, sched=newton_sched())
    for s in range(4):
        P.accumulate_factors(b, orc.random_matrix(m, n, 70 + s), cfg)
    for step, extra in ((3, 0), (6, 3)):
        for s in range(extra):
            P.accumulate_factors(b, orc.random_matrix(m, n, 80 + s), cfg)
        P.refresh_inverse(b, cfg, step)
        o = orc.Block(m, n, method)
        o.set(abi.FACTOR_L, b.factor_l)
        o.set(abi.FACTOR_R, b.factor_r)
        orc.refresh_inverse(o, cfg, step)
        errs = [rel(b.inv_l, o.inv_l), rel(b.inv_r, o.inv_r)]
        if method == abi.KL_SHAMPOO:
            errs += [rel(b.get(abi.KL_INV_L), o.get(abi.KL_INV_L)), rel(b.get(abi.KL_INV_R), o.get(abi.KL_INV_R))]
        print(m, n, abi.METHOD_NAMES[method], step, ["%.2e" % e for e in errs])
        assert max(errs) < 2e-5, errs
    assert b.version == 2


@pytest.mark.parametrize("precision", PRECS)
@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
def test_newton_refresh_kat(P, method, precision):
    """precond_test.cpp:107-121: the refresh of I is I; of 16 I is 0.5 I for
    L^-1/4 (Shampoo) and 0.25 I for L^-1/2 (KL-Shampoo); damping 0."""
    cfg = P.defaults_for(method)
    cfg.damping = 0.0
    b = P.PrecondBlock(4, 4, method, cfg, precision=precision, sched=newton_sched())
    b.set(abi.FACTOR_L, np.eye(4))
    b.set(abi.FACTOR_R, 16.0 * np.eye(4))
    P.refresh_inverse(b, cfg, 0)
    assert np.abs(b.inv_l - np.eye(4)).max() < 1e-6
    want = 0.5 if method == abi.SHAMPOO else 0.25
    assert np.abs(b.inv_r - want * np.eye(4)).max() < 1e-6


@pytest.mark.parametrize("precision", PRECS)
@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
def test_newton_rejects_indefinite(P, method, precision):
    """densela_test.cpp:110-115 (inv_root of an indefinite matrix -> NotPsd):
    a negative damped eigenvalue makes the iteration diverge, reported as
    NotPsdError at install (3XF16: the broken bounds overflow to inf, reported
    the same way)."""
    cfg = P.defaults_for(method)
    cfg.damping = 0.0
    b = P.PrecondBlock(2, 2, method, cfg, precision=precision, sched=newton_sched())
    b.set(abi.FACTOR_L, np.diag([1.0, -2.0]))
    b.set(abi.FACTOR_R, np.eye(2))
    with pytest.raises(abi.NotPsdError):
        P.refresh_inverse(b, cfg, 0)


@pytest.mark.parametrize("precision", PRECS)
@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
def test_newton_trajectory_matches_oracle_bounded_staleness(method, precision):
    """The trajectory case of test_gpu_step.py (three shape groups incl. a
    padded one, a 1-D AdamW parameter, pf=4, S=3, 2-step jobs) with the
    NEWTON refresh."""
    import test_gpu_step as T
    from paper_2605_16184_b200 import optimizer
    shapes = [(256, 384), (300,), (96, 96), (72, 72)]
    errs, o = T.run_pair(optimizer, method, shapes, limit=128, pf=4, steps=10, S=3, delay=2.0,
                         refresh_mode=abi.REFRESH_NEWTON, r_scale=2.5, precision=precision)
    assert o.stats().installed >= 2 * 8
    assert max(errs) <= 1.0, errs
