# SPDX-License-Identifier: Apache-2.0
"""Pins oracle/orc_np.py (the LAPACK-backed restatement used for the
large-block GPU parity tests) to the C oracle at the reference's own test
sizes: every method, Sum and EMA, cold start, refresh cadence, SOAP
re-projection, a rectangular block; relative agreement <= 1e-10 (the
reference's fp64 trajectory bound, harness_test.cpp:226-242), 1e-8 for SOAP's
update (eigenvector-sensitive, see below)."""
import numpy as np
import pytest

import orc
import orc_np
from paper_2605_16184_b200 import abi


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.SOAP, abi.KL_SHAMPOO])
@pytest.mark.parametrize("accum", [abi.SUM, abi.EMA])
@pytest.mark.parametrize("m,n", [(24, 24), (40, 17)])
def test_numpy_restatement_matches_c_oracle(method, accum, m, n):
    cfg = orc.defaults_for(method)
    cfg.accumulation = accum
    cfg.lr, cfg.weight_decay = 1e-2, 1e-3
    pf = 3
    ob, nb = orc.Block(m, n, method), orc_np.Block(m, n, method)
    th0 = orc.random_matrix(m, n, 5) * 0.1
    to, tn = th0.copy(), th0.copy()
    for step in range(9):
        # full-rank, separated spectra (eigenvector-sensitive SOAP stays well posed)
        q1 = np.linalg.qr(orc.random_matrix(m, m, 30 + step))[0]
        q2 = np.linalg.qr(orc.random_matrix(n, n, 40 + step))[0]
        k = min(m, n)
        g = 1e-2 * (q1[:, :k] * np.linspace(0.5, 1.5, k)) @ q2[:, :k].T
        orc.accumulate_factors(ob, g, cfg)
        orc_np.accumulate_factors(nb, g, cfg)
        if step % pf == pf - 1:  # first refresh once the factors are full rank (3 * 17 > 40)
            orc.refresh_inverse(ob, cfg, step)
            orc_np.refresh_inverse(nb, cfg, step)
        to = orc.apply_update(to, orc.step_update(ob, g, cfg), cfg)
        tn = orc_np.apply_update(tn, orc_np.step_update(nb, g, cfg), cfg)
    assert nb.version == ob.version == 3
    assert rel(nb.factor_l, ob.factor_l) < 1e-12
    assert rel(nb.factor_r, ob.factor_r) < 1e-12
    if method != abi.SOAP:
        assert rel(nb.inv_l, ob.inv_l) < 1e-10
        assert rel(nb.inv_r, ob.inv_r) < 1e-10
    if method == abi.KL_SHAMPOO:
        assert rel(nb.kl_inv_l, ob.get(abi.KL_INV_L)) < 1e-10
    if method == abi.SOAP:
        assert rel(nb.vals_l, ob.get(abi.EIGVALS_L)) < 1e-12
        # moments live in the (sign-ambiguous) rotated basis: compare Q M Q^T
        assert rel(nb.basis_l @ nb.rotated_m @ nb.basis_r.T, ob.basis_l @ ob.rotated_m @ ob.basis_r.T) < 1e-10
    # SOAP rotates into the basis: the C oracle's Jacobi stops at off(A) <= 1e-12 ||A||_F
    # (densela.hpp:192-203), so its eigenvectors carry ~1e-12 / relative gap
    assert rel(tn - th0, to - th0) < (1e-8 if method == abi.SOAP else 1e-10)
