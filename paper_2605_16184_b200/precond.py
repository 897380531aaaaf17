# SPDX-License-Identifier: Apache-2.0
"""Host-side mirror of the reference's per-block optimizer API
(proj/include/asopt/precond.hpp) over the C-ABI, with GPU-resident state.

Same names, argument meaning and error classes as the reference, so parity
tests read like proj/tests/precond_test.cpp. Matrices cross the boundary as
float64 numpy arrays; inside, state is fp32 (3xTF32 tensor-core products)
and the refresh eigendecomposition is fp64.

A ``PrecondBlock`` here owns a one-block blockset on the GPU. Its optimizer
configuration is bound at creation (the GPU kernels specialise on it);
functions that take ``cfg`` check it against the bound one.
"""
import ctypes as C

import numpy as np

from . import abi
from .runtime import check, lib, optimizer_defaults, partition_param  # noqa: F401  (re-export)

OptimizerConfig = abi.OptimizerConfig


def defaults_for(method):
    """OptimizerConfig::defaults_for (precond.cpp:44-62)."""
    return optimizer_defaults(method)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


_CFG_FIELDS = ("method", "accumulation", "beta1", "beta2", "eps", "damping")


class PrecondBlock:
    """PrecondBlock (precond.hpp:63-75) held in HBM."""

    def __init__(self, rows, cols, method, cfg=None, precision=abi.PREC_3XTF32, device=0, sched=None):
        import torch  # device memory for the (unused) parameter/gradient bindings
        self.rows, self.cols, self.method = int(rows), int(cols), int(method)
        self.cfg = (cfg.copy() if cfg is not None else defaults_for(method))
        self.cfg.method = method
        self.cfg.block_dim_limit = max(self.cfg.block_dim_limit, self.rows, self.cols)
        s = sched.copy() if sched is not None else abi.scheduler_defaults()
        s.pf = self.cfg.precondition_frequency
        self._theta = torch.zeros(self.rows, self.cols, dtype=torch.float32, device=f"cuda:{device}")
        self._grad = torch.zeros_like(self._theta)
        pd = abi.ParamDesc(self._theta.data_ptr(), self._grad.data_ptr(), self.rows, self.cols, self.cols, self.cols)
        h = C.c_void_p()
        check(lib.asg_blockset_create(device, C.byref(self.cfg), C.byref(s), C.byref(pd), 1, precision, 0, 1, 99,
                                      C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.asg_blockset_destroy(self._h)
            self._h = None

    # -- state access ---------------------------------------------------------
    def _shape(self, role):
        m, n = self.rows, self.cols
        return {abi.FACTOR_L: (m, m), abi.FACTOR_R: (n, n), abi.INV_L: (m, m), abi.INV_R: (n, n),
                abi.BASIS_L: (m, m), abi.BASIS_R: (n, n), abi.ROTATED_M: (m, n), abi.ROTATED_V: (m, n),
                abi.KL_INV_L: (m, m), abi.KL_INV_R: (n, n), abi.EIGVALS_L: (m,), abi.EIGVALS_R: (n,)}[role]

    def get(self, role):
        out = np.empty(self._shape(role))
        check(lib.asg_block_read(self._h, 0, role, _p(out), out.size))
        return out

    def set(self, role, value):
        v = _f64(value).reshape(self._shape(role))
        check(lib.asg_block_write(self._h, 0, role, _p(v), v.size))

    def info(self):
        i = abi.BlockInfo()
        check(lib.asg_blockset_block_info(self._h, 0, C.byref(i)))
        return i

    @property
    def version(self):
        return self.info().version

    @property
    def last_refresh_step(self):
        return self.info().last_refresh_step

    @property
    def moment_steps(self):
        return self.info().moment_steps

    def set_counters(self, version, last_refresh_step=-1, moment_steps=0):
        check(lib.asg_block_set_counters(self._h, 0, version, last_refresh_step, moment_steps))

    factor_l = property(lambda s: s.get(abi.FACTOR_L))
    factor_r = property(lambda s: s.get(abi.FACTOR_R))
    inv_l = property(lambda s: s.get(abi.INV_L))
    inv_r = property(lambda s: s.get(abi.INV_R))
    basis_l = property(lambda s: s.get(abi.BASIS_L))
    basis_r = property(lambda s: s.get(abi.BASIS_R))
    rotated_m = property(lambda s: s.get(abi.ROTATED_M))
    rotated_v = property(lambda s: s.get(abi.ROTATED_V))


def _check_cfg(b, cfg):
    if cfg is None:
        return
    for f in _CFG_FIELDS:
        if getattr(cfg, f) != getattr(b.cfg, f):
            raise abi.InvalidArgumentError(f"cfg.{f} differs from the block's bound configuration")


def _shape_check(b, g, what):
    if g.shape != (b.rows, b.cols):
        raise abi.ShapeMismatchError(f"{what}: gradient shape mismatch")


def accumulate_factors(b, g, cfg=None):
    """accumulate_factors (precond.cpp:173-189)."""
    _check_cfg(b, cfg)
    g = _f64(g)
    _shape_check(b, g, "accumulate_factors")
    check(lib.asg_block_accumulate_f64(b._h, 0, _p(g), g.shape[1]))


def refresh_inverse(b, cfg=None, step=0):
    """In place: install_refresh(b, compute_refresh(snapshot_factors(b), cfg), step)
    (precond.cpp:166-171); the eigendecomposition runs on the GPU in fp64."""
    _check_cfg(b, cfg)
    check(lib.asg_block_refresh_f64(b._h, 0, step))


def precondition_shampoo(b, g):
    """precondition_shampoo (precond.cpp:191-198); for KL-Shampoo blocks this is
    L^-1/2 G R^-1/2 with the installed roots."""
    g = _f64(g)
    _shape_check(b, g, "precondition_shampoo")
    out = np.empty_like(g)
    check(lib.asg_block_precondition_f64(b._h, 0, _p(g), g.shape[1], _p(out)))
    return out


def soap_scaled_step(b, g, cfg=None):
    """soap_scaled_step (precond.cpp:208-223)."""
    _check_cfg(b, cfg)
    g = _f64(g)
    _shape_check(b, g, "precondition_soap")
    out = np.empty_like(g)
    check(lib.asg_block_soap_step_f64(b._h, 0, _p(g), g.shape[1], _p(out)))
    return out


def precondition_soap(b, g, cfg=None):
    """precondition_soap (precond.cpp:200-206)."""
    if b.version == 0:
        raise abi.StaleUninitializedError("precondition_soap: no basis installed")
    return soap_scaled_step(b, g, cfg)


# ---- the split refresh (precond.hpp:77-98) --------------------------------------
class FactorSnapshot:
    """snapshot_factors (precond.cpp:112-117): device copies of L and R."""

    def __init__(self, handle):
        self._h = handle

    @property
    def checksum(self):
        """snapshot_checksum (precond.cpp:114-115) over the fp32 factor bytes."""
        v = C.c_uint64()
        check(lib.asg_snapshot_checksum(self._h, C.byref(v)))
        return v.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib.asg_snapshot_destroy(self._h)
            self._h = None


class RefreshResult:
    """compute_refresh's result (precond.hpp:83-87), held in HBM until installed."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None):
            lib.asg_refresh_result_destroy(self._h)
            self._h = None


def snapshot_factors(b):
    h = C.c_void_p()
    check(lib.asg_snapshot_factors(b._h, 0, C.byref(h)))
    return FactorSnapshot(h)


def compute_refresh(b, snap, cfg=None):
    """Pure over the snapshot (precond.cpp:129-142); computed with the
    block's refresh arithmetic."""
    _check_cfg(b, cfg)
    h = C.c_void_p()
    check(lib.asg_compute_refresh(b._h, snap._h, C.byref(h)))
    return RefreshResult(h)


def install_refresh(b, result, step):
    """install_refresh (precond.cpp:144-164); consumes the result."""
    h, result._h = result._h, None
    check(lib.asg_install_refresh(b._h, 0, h, step))


def replicated_state(b):
    """replicated_state (precond.cpp:253-265): [L side | R side] of the inverse
    roots (Shampoo / KL-Shampoo) or the eigenbases (SOAP)."""
    out = np.empty(b.rows * b.rows + b.cols * b.cols)
    check(lib.asg_block_replicated_state(b._h, 0, _p(out), out.size))
    return out


def load_replicated_state(b, flat):
    """load_replicated_state (precond.cpp:267-279)."""
    flat = _f64(flat).ravel()
    check(lib.asg_block_load_replicated_state(b._h, 0, _p(flat), flat.size))


class AdamState:
    """AdamState (precond.hpp:122-126) with its moments in HBM."""

    def __init__(self, rows, cols):
        self.shape = (rows, cols)
        h = C.c_void_p()
        check(lib.asg_adam_state_create(rows, cols, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.asg_adam_state_destroy(self._h)
            self._h = None


def adamw_step(state, g, cfg):
    """adamw_step (precond.cpp:229-242): the bias-corrected Adam direction."""
    g = _f64(g)
    if g.shape != state.shape:
        raise abi.ShapeMismatchError("adamw_step: gradient shape mismatch")
    out = np.empty_like(g)
    check(lib.asg_adamw_step_f64(state._h, _p(g), C.byref(cfg), _p(out)))
    return out


def apply_update(theta, update, cfg, lr_scale=1.0):
    """apply_update (precond.cpp:244-251); returns the updated copy of theta."""
    t = _f64(theta).copy()
    u = _f64(update)
    if t.shape != u.shape:
        raise abi.ShapeMismatchError("apply_update: shape mismatch")
    check(lib.asg_apply_update_f64(_p(t), _p(u), t.shape[0], t.shape[1] if t.ndim > 1 else 1, C.byref(cfg), lr_scale))
    return t
