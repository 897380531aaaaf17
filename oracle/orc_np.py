# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY: LAPACK-backed numpy restatement of the oracle's
per-block path, for parity checks at block dimensions (1024, 2048) where the
oracle's cyclic Jacobi (densela.hpp:182-264, restated in asteria_oracle.cpp)
takes minutes per factor on one core.

It follows oracle/asteria_oracle.cpp function by function (each cites the
reference line it restates) with one substitution: sym_eig is
numpy.linalg.eigh (LAPACK syevd). The result of the reference's eigensolver
does not depend on the algorithm beyond its tolerance (off(A) <= 1e-12
||A||_F, densela.hpp:192-203): values ascending, vectors as columns; the
eigenvector signs differ, which every quantity on the path is invariant to
(roots; SOAP updates and the re-projection rot = Q_new^T Q_old, where a sign
flip of a basis vector flips the matching moment row and cancels).
tests/test_oracle_np.py pins this restatement to the C oracle at the
reference's test sizes (<= 1e-10), so the large-n checks inherit the oracle's
pinning (tests/test_oracle_*.py against the reference's known answers).

Only tests/ may import this module.
"""
import numpy as np

from paper_2605_16184_b200 import abi


def symmetrized(p):  # densela.hpp:152-156
    return 0.5 * (p + p.T)


def sym_eig(a):  # densela.hpp:182-264 (values ascending, vectors as columns)
    w, v = np.linalg.eigh(symmetrized(np.asarray(a, dtype=np.float64)))
    return w, v


def relative_damping(m, damping):  # precond.cpp:121-125
    n = m.shape[0]
    return damping * np.trace(m) / n if n else 0.0


def reconstruct(w, v, f):  # densela.hpp:280 (V diag(f) V^T, symmetrized)
    return symmetrized((v * f) @ v.T)


def inv_root(a, p, eps):  # densela.hpp:267-282
    w, v = sym_eig(a)
    d = w + eps
    if np.any(d <= 0):
        raise abi.NotPsdError("inv_root: damped eigenvalue <= 0")
    return reconstruct(w, v, d ** (-1.0 / p))


class Block:
    """PrecondBlock (precond.hpp:63-75; create precond.cpp:84-110). KL-Shampoo
    starts from identity statistics (asteria_oracle.cpp Block::create)."""

    def __init__(self, rows, cols, method):
        self.rows, self.cols, self.method = rows, cols, method
        kl = method == abi.KL_SHAMPOO
        self.factor_l = np.eye(rows) if kl else np.zeros((rows, rows))
        self.factor_r = np.eye(cols) if kl else np.zeros((cols, cols))
        self.inv_l, self.inv_r = np.eye(rows), np.eye(cols)
        self.kl_inv_l, self.kl_inv_r = np.eye(rows), np.eye(cols)
        self.basis_l, self.basis_r = np.eye(rows), np.eye(cols)
        self.vals_l, self.vals_r = np.ones(rows), np.ones(cols)
        self.rotated_m = np.zeros((rows, cols))
        self.rotated_v = np.zeros((rows, cols))
        self.version, self.last_refresh_step, self.moment_steps = 0, -1, 0


def accumulate_factors(b, g, cfg):  # precond.cpp:173-189 (+ KL statistics)
    g = np.asarray(g, dtype=np.float64)
    if not np.all(np.isfinite(g)):
        raise abi.NonFiniteError("accumulate_factors: non-finite gradient")
    if b.method == abi.KL_SHAMPOO:
        gl = symmetrized(g @ b.kl_inv_r @ g.T) / b.cols
        gr = symmetrized(g.T @ b.kl_inv_l @ g) / b.rows
    else:
        gl, gr = symmetrized(g @ g.T), symmetrized(g.T @ g)  # gram_left/right densela.hpp:160-175
    if cfg.accumulation == abi.SUM:
        b.factor_l = b.factor_l + gl
        b.factor_r = b.factor_r + gr
    else:
        beta = cfg.beta2
        b.factor_l = beta * b.factor_l + (1.0 - beta) * gl
        b.factor_r = beta * b.factor_r + (1.0 - beta) * gr


def compute_refresh(fl, fr, cfg):  # precond.cpp:129-142 (+ KL: L^-1/2 and L^-1)
    if cfg.method == abi.SOAP:
        return {"soap": sym_eig(fl) + sym_eig(fr)}
    if cfg.method == abi.KL_SHAMPOO:
        out = {}
        for side, f in (("l", fl), ("r", fr)):
            w, v = sym_eig(f)
            d = w + relative_damping(f, cfg.damping)
            if np.any(d <= 0):
                raise abi.NotPsdError("kl refresh: damped eigenvalue <= 0")
            out["inv_" + side] = reconstruct(w, v, d ** -0.5)
            out["kl_inv_" + side] = reconstruct(w, v, 1.0 / d)
        return out
    return {"inv_l": inv_root(fl, 4, relative_damping(fl, cfg.damping)),
            "inv_r": inv_root(fr, 4, relative_damping(fr, cfg.damping))}


def install_refresh(b, r, step):  # precond.cpp:144-164
    if "soap" in r:
        wl, ql, wr, qr = r["soap"]
        rot_l, rot_r = ql.T @ b.basis_l, qr.T @ b.basis_r
        b.rotated_m = rot_l @ b.rotated_m @ rot_r.T
        b.rotated_v = (rot_l * rot_l) @ b.rotated_v @ (rot_r * rot_r).T
        b.basis_l, b.basis_r, b.vals_l, b.vals_r = ql, qr, wl, wr
    else:
        for k, val in r.items():
            setattr(b, k, val)
    b.version += 1
    b.last_refresh_step = step


def refresh_inverse(b, cfg, step):  # precond.cpp:166-171
    install_refresh(b, compute_refresh(b.factor_l.copy(), b.factor_r.copy(), cfg), step)


def soap_scaled_step(b, g, cfg):  # precond.cpp:208-223
    rotated = b.basis_l.T @ g @ b.basis_r
    b.moment_steps += 1
    t = float(b.moment_steps)
    b.rotated_m = cfg.beta1 * b.rotated_m + (1.0 - cfg.beta1) * rotated
    b.rotated_v = cfg.beta2 * b.rotated_v + (1.0 - cfg.beta2) * rotated * rotated
    m_hat = b.rotated_m / (1.0 - cfg.beta1 ** t)
    v_hat = b.rotated_v / (1.0 - cfg.beta2 ** t)
    return b.basis_l @ (m_hat / (np.sqrt(v_hat) + cfg.eps)) @ b.basis_r.T


def step_update(b, g, cfg):  # cold-start rule harness.cpp:455-466 + precondition_* precond.cpp:191-223
    g = np.asarray(g, dtype=np.float64)
    if b.method == abi.SOAP:
        return soap_scaled_step(b, g, cfg)
    if b.version == 0:
        return g
    return b.inv_l @ g @ b.inv_r


def apply_update(theta, update, cfg, lr_scale=1.0):  # precond.cpp:244-251
    if not np.all(np.isfinite(update)):
        raise abi.NonFiniteError("apply_update: non-finite update")
    return theta - cfg.lr * lr_scale * (update + cfg.weight_decay * theta)
