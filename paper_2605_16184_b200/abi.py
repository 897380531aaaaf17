# SPDX-License-Identifier: Apache-2.0
"""ctypes mirror of include/asteria_b200.h (structs, enums, status codes).

The exception classes carry the reference's names (proj/include/asopt/errors.hpp:10-47)
so code written against the reference's error taxonomy ports unchanged.
"""
import ctypes as C

ASG_OK = 0

# asg_method (precond.hpp:19 + KL-Shampoo)
ADAMW, SHAMPOO, SOAP, KL_SHAMPOO = 0, 1, 2, 3
METHOD_NAMES = {ADAMW: "AdamW", SHAMPOO: "Shampoo", SOAP: "SOAP", KL_SHAMPOO: "KL-Shampoo"}
# asg_accumulation (precond.hpp:20)
SUM, EMA = 0, 1
# asg_precision
PREC_3XTF32, PREC_TF32, PREC_3XTF32_SMEM, PREC_3XF16 = 0, 1, 2, 3
# asg_install_mode
INSTALL_SIM_CLOCK, INSTALL_EVENT = 0, 1
# asg_refresh_mode
REFRESH_F64, REFRESH_F32, REFRESH_NEWTON = 0, 1, 2
# asg_role (tiers.hpp:35-44 + KL + eigenvalues)
(FACTOR_L, FACTOR_R, INV_L, INV_R, BASIS_L, BASIS_R, ROTATED_M, ROTATED_V,
 KL_INV_L, KL_INV_R, EIGVALS_L, EIGVALS_R) = range(12)
# asg_event_kind
(EV_DISPATCH, EV_JOB_START, EV_JOB_DONE, EV_INSTALL, EV_BARRIER_WAIT_BEGIN, EV_BARRIER_WAIT_END,
 EV_PREFETCH, EV_DRAIN) = range(8)
# asg_hook (HookEvent::Kind asyncsched.hpp)
HOOK_FORWARD_POST, HOOK_BACKWARD_PRE, HOOK_STEP_END = range(3)


class OptimizerConfig(C.Structure):
    """asg_optimizer_config == asopt::OptimizerConfig (precond.hpp:27-44)."""
    _fields_ = [
        ("method", C.c_int32),
        ("accumulation", C.c_int32),
        ("lr", C.c_double),
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("eps", C.c_double),
        ("weight_decay", C.c_double),
        ("precondition_frequency", C.c_int64),
        ("damping", C.c_double),
        ("block_dim_limit", C.c_int64),
    ]

    def copy(self):
        c = OptimizerConfig()
        C.pointer(c)[0] = self
        return c

    def __repr__(self):
        return "OptimizerConfig(" + ", ".join(f"{n}={getattr(self, n)!r}" for n, _ in self._fields_) + ")"


class SchedulerConfig(C.Structure):
    """asg_scheduler_config == asopt::SchedulerConfig (asyncsched.hpp:50-59)."""
    _fields_ = [
        ("staleness_S", C.c_int64),
        ("pf", C.c_int64),
        ("pool_size", C.c_int32),
        ("drain_budget", C.c_int32),
        ("inject_job_delay_steps", C.c_double),
        ("inject_job_delay_jitter_steps", C.c_double),
        ("step_compute_us", C.c_double),
        ("install_cost_us", C.c_double),
        ("install_mode", C.c_int32),
        ("refresh_mode", C.c_int32),
    ]

    def copy(self):
        c = SchedulerConfig()
        C.pointer(c)[0] = self
        return c


def scheduler_defaults():
    """SchedulerConfig{} defaults (asyncsched.hpp:50-59)."""
    s = SchedulerConfig()
    s.staleness_S, s.pf, s.pool_size, s.drain_budget = 5, 10, 0, 4
    s.inject_job_delay_steps, s.inject_job_delay_jitter_steps = 0.0, 0.0
    s.step_compute_us, s.install_cost_us = 1000.0, 0.0
    s.install_mode = INSTALL_SIM_CLOCK
    s.refresh_mode = REFRESH_F64
    return s


class BlockSpec(C.Structure):
    """asg_block_spec == asopt::BlockSpec (precond.hpp:47-57)."""
    _fields_ = [
        ("param_index", C.c_int64),
        ("row_begin", C.c_int64),
        ("row_end", C.c_int64),
        ("col_begin", C.c_int64),
        ("col_end", C.c_int64),
        ("block_dim_limit", C.c_int64),
    ]

    def rows(self):
        return self.row_end - self.row_begin

    def cols(self):
        return self.col_end - self.col_begin

    def id(self, param_id="w"):
        """BlockSpec::id (precond.cpp:64-67)."""
        return f"{param_id}[{self.row_begin}:{self.row_end},{self.col_begin}:{self.col_end}]"


class ParamDesc(C.Structure):
    _fields_ = [
        ("theta", C.c_void_p),
        ("grad", C.c_void_p),
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("ld_theta", C.c_int64),
        ("ld_grad", C.c_int64),
    ]


class Freshness(C.Structure):
    """asg_freshness == asopt::FreshnessRecord (asyncsched.hpp:72-78)."""
    _fields_ = [
        ("installed_version", C.c_uint64),
        ("dispatch_step_of_pending", C.c_int64),
        ("last_install_step", C.c_int64),
        ("installed_snapshot_step", C.c_int64),
    ]


class PoolStats(C.Structure):
    """asg_pool_stats == asopt::PoolStats (asyncsched.hpp:61-70)."""
    _fields_ = [
        ("dispatched", C.c_uint64),
        ("completed", C.c_uint64),
        ("installed", C.c_uint64),
        ("coalesced", C.c_uint64),
        ("barrier_waits", C.c_uint64),
        ("wait_total_us", C.c_double),
        ("pending", C.c_int32),
        ("queue_depth", C.c_int32),
    ]


class BlockInfo(C.Structure):
    _fields_ = [
        ("spec", BlockSpec),
        ("version", C.c_uint64),
        ("last_refresh_step", C.c_int64),
        ("moment_steps", C.c_int64),
        ("owner_rank", C.c_int32),
        ("use_adamw", C.c_int32),
    ]


class Event(C.Structure):
    _fields_ = [
        ("step", C.c_int64),
        ("kind", C.c_int32),
        ("reserved", C.c_int32),
        ("block", C.c_int64),
        ("version", C.c_uint64),
        ("t_us", C.c_double),
    ]


HBM_PREP, HBM_SQNORM, HBM_ADAMW, HBM_KINDS = 0, 1, 2, 3
HBM_NAMES = {HBM_PREP: "prep", HBM_SQNORM: "sqnorm", HBM_ADAMW: "adamw"}


class HbmStats(C.Structure):
    _fields_ = [("launches", C.c_uint64 * HBM_KINDS), ("bytes", C.c_double * HBM_KINDS),
                ("ms", C.c_double * HBM_KINDS)]


class KernelStats(C.Structure):
    _fields_ = [
        ("launches", C.c_uint64),
        ("gemm_launches", C.c_uint64),
        ("gemm_alg_flops", C.c_double),
        ("gemm_ms", C.c_double),
    ]


# ---- error taxonomy (errors.hpp:10-47) --------------------------------------
class Error(RuntimeError):
    code = -1


class NonFiniteError(Error):
    code = 1


class NoConvergenceError(Error):
    code = 2


class NotPsdError(Error):
    code = 3


class LayoutMismatchError(Error):
    code = 4


class ShapeMismatchError(Error):
    code = 5


class StaleUninitializedError(Error):
    code = 6


class WorkerPoolDownError(Error):
    code = 7


class ConfigInvalidError(Error):
    code = 8


class AuditError(Error):
    code = 9


class MissingKeyError(Error):
    code = 10


class CudaError(Error):
    code = 11


class OutOfMemoryError(Error):
    code = 12


class InvalidArgumentError(Error):
    code = 13


class UnsupportedError(Error):
    code = 14


class CapacityExhaustedError(Error):
    code = 15


class IoError(Error):
    code = 16


class PinnedEntryError(Error):
    code = 17


class DirtyNotPersistedError(Error):
    code = 18


_BY_CODE = {cls.code: cls for cls in (
    NonFiniteError, NoConvergenceError, NotPsdError, LayoutMismatchError, ShapeMismatchError,
    StaleUninitializedError, WorkerPoolDownError, ConfigInvalidError, AuditError,
    MissingKeyError, CudaError, OutOfMemoryError, InvalidArgumentError, UnsupportedError,
    CapacityExhaustedError, IoError, PinnedEntryError, DirtyNotPersistedError)}


# ---- tiered store (F3; tierstore.hpp) ----------------------------------------
TIER_HOT, TIER_HOST, TIER_COLD = 0, 1, 2
TIER_NAMES = {TIER_HOT: "Hot", TIER_HOST: "Host", TIER_COLD: "Cold"}


class StoreConfig(C.Structure):
    _fields_ = [("hot_capacity_bytes", C.c_uint64), ("host_capacity_bytes", C.c_uint64),
                ("cold_path", C.c_char_p), ("transfer_bandwidth_bytes_per_sec", C.c_double),
                ("transfer_latency_us", C.c_uint64), ("hot_device", C.c_int32)]


class EntryView(C.Structure):
    _fields_ = [("tier", C.c_int32), ("bytes", C.c_uint64), ("dirty", C.c_int32), ("pinned", C.c_int32),
                ("last_touch_step", C.c_int64), ("staged_pending", C.c_int32), ("staged_ready", C.c_int32)]


class Residency(C.Structure):
    _fields_ = [("hot_bytes", C.c_uint64), ("host_bytes", C.c_uint64), ("cold_bytes", C.c_uint64)]


class IoCounters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "file_writes", "file_reads", "write_skips", "page_ins", "evictions", "prefetch_requests",
        "transfers_started", "transfers_coalesced", "transfers_completed", "transfers_dropped",
        "drains_installed")]


def raise_for(code, message):
    """Maps an asg_status to the matching exception class."""
    if code == ASG_OK:
        return
    raise _BY_CODE.get(code, Error)(message)
