# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY: numpy/ctypes front-end of the CPU oracle (liborc.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may use
this module, as the checker or the timed CPU baseline. The product package
(paper_2605_16184_b200) never imports it.

Every function restates a reference function; see oracle/asteria_oracle.cpp
for the file:line citations.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2605_16184_b200 import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liborc.so")
_lib = None

_dp = C.POINTER(C.c_double)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


NATIVE_PATH = os.path.join("/tmp", "asg_oracle_native", "liborc_native.so")


def use_build(native=False):
    """Selects the -O3 build (the reference's Release flags) or an
    -O3 -march=native one compiled on this machine (make native) for
    subsequent calls; objects created under one build must not be passed to
    the other."""
    global _lib, _LIB_PATH
    path = NATIVE_PATH if native else os.path.join(_HERE, "build", "liborc.so")
    if native and not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", _HERE, "native", f"NATIVE={path}"], check=True)
    if path != _LIB_PATH:
        _LIB_PATH, _lib = path, None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        for name in ("orc_block_create", "orc_block_clone", "orc_adam_create", "orc_sched_create"):
            getattr(L, name).restype = C.c_void_p
        L.orc_block_create.argtypes = [C.c_int64, C.c_int64, C.c_int]
        L.orc_block_clone.argtypes = [C.c_void_p]
        L.orc_block_free.argtypes = [C.c_void_p]
        L.orc_adam_create.argtypes = [C.c_int64, C.c_int64]
        L.orc_adam_free.argtypes = [C.c_void_p]
        L.orc_sched_create.argtypes = [C.POINTER(abi.OptimizerConfig), C.POINTER(abi.SchedulerConfig), C.c_uint64]
        L.orc_sched_free.argtypes = [C.c_void_p]
        L.orc_clip_scale.restype = C.c_double
        L.orc_clip_scale.argtypes = [_dp, C.c_int64, C.c_double]
        L.orc_warmup_scale.restype = C.c_double
        L.orc_warmup_scale.argtypes = [C.c_int64, C.c_int64]
        L.orc_sched_events.restype = C.c_int64
        L.orc_sched_clock_advance.argtypes = [C.c_void_p, C.c_double]
        _lib = L
    return _lib


def _check(code):
    if code != abi.ASG_OK:
        abi.raise_for(code, lib().orc_last_error().decode())


def _p(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- densela ----------------------------------------------------------------
def random_matrix(rows, cols, seed):
    """test_util.hpp:10-17 (mt19937_64 + std::normal_distribution)."""
    out = np.empty((rows, cols))
    _check(lib().orc_random_matrix(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), _p(out)))
    return out


def random_spd(dim, seed, ridge=1e-3):
    """test_util.hpp:20-26."""
    out = np.empty((dim, dim))
    _check(lib().orc_random_spd(C.c_int64(dim), C.c_uint64(seed), C.c_double(ridge), _p(out)))
    return out


def gram_left(g):
    g = _f64(g)
    out = np.empty((g.shape[0], g.shape[0]))
    _check(lib().orc_gram_left(_p(g), C.c_int64(g.shape[0]), C.c_int64(g.shape[1]), _p(out)))
    return out


def gram_right(g):
    g = _f64(g)
    out = np.empty((g.shape[1], g.shape[1]))
    _check(lib().orc_gram_right(_p(g), C.c_int64(g.shape[0]), C.c_int64(g.shape[1]), _p(out)))
    return out


def sym_eig(a):
    """densela.hpp:182-264: (values ascending, vectors as columns)."""
    a = _f64(a)
    n = a.shape[0]
    vals, vecs = np.empty(n), np.empty((n, n))
    _check(lib().orc_sym_eig(_p(a), C.c_int64(n), _p(vals), _p(vecs)))
    return vals, vecs


def inv_root(a, root_order, damping):
    """densela.hpp:267-282."""
    a = _f64(a)
    n = a.shape[0]
    out = np.empty((n, n))
    _check(lib().orc_inv_root(_p(a), C.c_int64(n), C.c_int(root_order), C.c_double(damping), _p(out)))
    return out


def inv_root_xp(a, root_order, damping):
    """test_util.hpp:32-37: same algorithm in long double."""
    a = _f64(a)
    n = a.shape[0]
    out = np.empty((n, n))
    _check(lib().orc_inv_root_xp(_p(a), C.c_int64(n), C.c_int(root_order), C.c_double(damping), _p(out)))
    return out


def pack_spd(a):
    a = _f64(a)
    n = a.shape[0]
    out = np.empty(n * (n + 1) // 2)
    _check(lib().orc_pack_spd(_p(a), C.c_int64(n), _p(out)))
    return out


def unpack_spd(p, n):
    p = _f64(p)
    out = np.empty((n, n))
    _check(lib().orc_unpack_spd(_p(p), C.c_int64(n), _p(out)))
    return out


def checksum(a):
    a = _f64(a)
    out = C.c_uint64()
    _check(lib().orc_checksum(_p(a), C.c_int64(a.size), C.byref(out)))
    return out.value


# ---- precond ------------------------------------------------------------------
def defaults_for(method):
    c = abi.OptimizerConfig()
    _check(lib().orc_defaults_for(C.c_int(method), C.byref(c)))
    return c


def validate(cfg):
    _check(lib().orc_validate(C.byref(cfg)))


_ROLE_SHAPE = {
    abi.FACTOR_L: "mm", abi.FACTOR_R: "nn", abi.INV_L: "mm", abi.INV_R: "nn",
    abi.BASIS_L: "mm", abi.BASIS_R: "nn", abi.ROTATED_M: "mn", abi.ROTATED_V: "mn",
    abi.KL_INV_L: "mm", abi.KL_INV_R: "nn", abi.EIGVALS_L: "m", abi.EIGVALS_R: "n",
}


class Block:
    """PrecondBlock (precond.hpp:63-75) held by the oracle."""

    def __init__(self, rows, cols, method, _handle=None):
        self.rows, self.cols, self.method = rows, cols, method
        self._h = _handle or lib().orc_block_create(C.c_int64(rows), C.c_int64(cols), C.c_int(method))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_block_free(C.c_void_p(self._h))
            self._h = None

    def clone(self):
        return Block(self.rows, self.cols, self.method, _handle=lib().orc_block_clone(C.c_void_p(self._h)))

    def _shape(self, role):
        s = _ROLE_SHAPE[role]
        dims = {"m": self.rows, "n": self.cols}
        return tuple(dims[ch] for ch in s)

    def get(self, role):
        out = np.empty(self._shape(role))
        _check(lib().orc_block_get(C.c_void_p(self._h), C.c_int(role), _p(out)))
        return out

    def set(self, role, value):
        v = _f64(value).reshape(self._shape(role))
        _check(lib().orc_block_set(C.c_void_p(self._h), C.c_int(role), _p(v)))

    def counters(self):
        v, l, m = C.c_uint64(), C.c_int64(), C.c_int64()
        lib().orc_block_counters(C.c_void_p(self._h), C.byref(v), C.byref(l), C.byref(m))
        return v.value, l.value, m.value

    def set_counters(self, version, last_refresh_step=-1, moment_steps=0):
        lib().orc_block_set_counters(C.c_void_p(self._h), C.c_uint64(version),
                                     C.c_int64(last_refresh_step), C.c_int64(moment_steps))

    @property
    def version(self):
        return self.counters()[0]

    @property
    def last_refresh_step(self):
        return self.counters()[1]

    @property
    def moment_steps(self):
        return self.counters()[2]

    factor_l = property(lambda s: s.get(abi.FACTOR_L))
    factor_r = property(lambda s: s.get(abi.FACTOR_R))
    inv_l = property(lambda s: s.get(abi.INV_L))
    inv_r = property(lambda s: s.get(abi.INV_R))
    basis_l = property(lambda s: s.get(abi.BASIS_L))
    basis_r = property(lambda s: s.get(abi.BASIS_R))
    rotated_m = property(lambda s: s.get(abi.ROTATED_M))
    rotated_v = property(lambda s: s.get(abi.ROTATED_V))

    def snapshot_checksum(self):
        out = C.c_uint64()
        _check(lib().orc_snapshot_checksum(C.c_void_p(self._h), C.byref(out)))
        return out.value


def accumulate_factors(b, g, cfg):
    g = _f64(g)
    _check(lib().orc_accumulate(C.c_void_p(b._h), _p(g), C.byref(cfg)))


def refresh_inverse(b, cfg, step):
    """In place: install_refresh(b, compute_refresh(snapshot_factors(b)), step)."""
    _check(lib().orc_refresh_inverse(C.c_void_p(b._h), C.byref(cfg), C.c_int64(step)))


def refresh_from(dst, src, cfg, step):
    _check(lib().orc_refresh_from(C.c_void_p(dst._h), C.c_void_p(src._h), C.byref(cfg), C.c_int64(step)))


def precondition_shampoo(b, g):
    g = _f64(g)
    out = np.empty_like(g)
    _check(lib().orc_precondition_shampoo(C.c_void_p(b._h), _p(g), _p(out)))
    return out


def precondition_soap(b, g, cfg):
    g = _f64(g)
    out = np.empty_like(g)
    _check(lib().orc_precondition_soap(C.c_void_p(b._h), _p(g), C.byref(cfg), _p(out)))
    return out


def soap_scaled_step(b, g, cfg):
    g = _f64(g)
    out = np.empty_like(g)
    _check(lib().orc_soap_scaled_step(C.c_void_p(b._h), _p(g), C.byref(cfg), _p(out)))
    return out


def step_update(b, g, cfg):
    """Cold-start rule + precondition (harness.cpp:455-466)."""
    g = _f64(g)
    out = np.empty_like(g)
    _check(lib().orc_step_update(C.c_void_p(b._h), _p(g), C.byref(cfg), _p(out)))
    return out


def apply_update(theta, update, cfg, lr_scale=1.0):
    """Returns the updated copy of theta (precond.cpp:244-251)."""
    t = _f64(theta).copy()
    u = _f64(update)
    _check(lib().orc_apply_update(_p(t), _p(u), C.c_int64(t.shape[0]), C.c_int64(t.shape[1]),
                                  C.byref(cfg), C.c_double(lr_scale)))
    return t


def replicated_state(b):
    out = np.empty(b.rows * b.rows + b.cols * b.cols)
    _check(lib().orc_replicated_state(C.c_void_p(b._h), _p(out)))
    return out


class AdamState:
    def __init__(self, rows, cols):
        self.shape = (rows, cols)
        self._h = lib().orc_adam_create(C.c_int64(rows), C.c_int64(cols))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_adam_free(C.c_void_p(self._h))
            self._h = None


def adamw_step(state, g, cfg):
    g = _f64(g)
    out = np.empty_like(g)
    _check(lib().orc_adamw_step(C.c_void_p(state._h), _p(g), C.byref(cfg), _p(out)))
    return out


def clip_scale(flat, clip_norm=1.0):
    f = _f64(flat).ravel()
    return lib().orc_clip_scale(_p(f), C.c_int64(f.size), C.c_double(clip_norm))


def warmup_scale(step, total):
    return lib().orc_warmup_scale(C.c_int64(step), C.c_int64(total))


def refresh_many(blocks, cfg, step, threads):
    arr = (C.c_void_p * len(blocks))(*[b._h for b in blocks])
    _check(lib().orc_refresh_many(arr, C.c_int64(len(blocks)), C.byref(cfg), C.c_int64(step), C.c_int(threads)))


# ---- scheduler ------------------------------------------------------------------
class Scheduler:
    """ShadowScheduler rules on a simulated clock (asyncsched.cpp:108-221,268-286)."""

    def __init__(self, opt, sched, seed=99):
        self._h = lib().orc_sched_create(C.byref(opt), C.byref(sched), C.c_uint64(seed))
        if not self._h:
            raise abi.ConfigInvalidError(lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_sched_free(C.c_void_p(self._h))
            self._h = None

    def advance(self, us):
        lib().orc_sched_clock_advance(C.c_void_p(self._h), C.c_double(us))

    def maybe_dispatch(self, block, bid, step):
        d = C.c_int()
        _check(lib().orc_sched_maybe_dispatch(C.c_void_p(self._h), C.c_void_p(block._h), C.c_int64(bid),
                                              C.c_int64(step), C.byref(d)))
        return bool(d.value)

    def staleness_barrier(self, block, bid, step):
        w = C.c_double()
        _check(lib().orc_sched_barrier(C.c_void_p(self._h), C.c_void_p(block._h), C.c_int64(bid),
                                       C.c_int64(step), C.byref(w)))
        return w.value

    def step_end(self, blocks, ids, step):
        arr = (C.c_void_p * len(blocks))(*[b._h for b in blocks])
        idarr = (C.c_int64 * len(ids))(*ids)
        _check(lib().orc_sched_step_end(C.c_void_p(self._h), arr, idarr, C.c_int64(len(blocks)), C.c_int64(step)))

    def stats(self):
        s = abi.PoolStats()
        lib().orc_sched_stats(C.c_void_p(self._h), C.byref(s))
        return s

    def freshness(self, bid):
        f = abi.Freshness()
        _check(lib().orc_sched_freshness(C.c_void_p(self._h), C.c_int64(bid), C.byref(f)))
        return f

    def events(self):
        n = lib().orc_sched_events(C.c_void_p(self._h), None, C.c_int64(0))
        buf = (abi.Event * max(1, n))()
        lib().orc_sched_events(C.c_void_p(self._h), buf, C.c_int64(n))
        return [buf[i] for i in range(n)]

    def stop_pool(self):
        lib().orc_sched_stop_pool(C.c_void_p(self._h))
