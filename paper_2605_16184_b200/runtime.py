# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the product library (include/asteria_b200.h).

Importing this module loads ``csrc/build/libasteria_b200.so`` and fails
loudly if it is missing: there is no CPU fallback anywhere in the product.
"""
import ctypes as C
import os

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "csrc", "build", "libasteria_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or `make -C paper_2605_16184_b200/csrc`). There is no CPU fallback.")

lib = C.CDLL(LIB_PATH)

_vp = C.c_void_p
_i32, _i64, _u64, _f32, _f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
_P = C.POINTER

_SIGS = {
    "asg_last_error": (C.c_char_p, []),
    "asg_api_version": (C.c_int, []),
    "asg_device_supported": (C.c_int, [C.c_int]),
    "asg_optimizer_defaults": (C.c_int, [_i32, _P(abi.OptimizerConfig)]),
    "asg_optimizer_validate": (C.c_int, [_P(abi.OptimizerConfig)]),
    "asg_scheduler_defaults": (C.c_int, [_P(abi.SchedulerConfig)]),
    "asg_config_from_json": (C.c_int, [C.c_char_p, _P(abi.OptimizerConfig), _P(abi.SchedulerConfig), _P(_i32)]),
    "asg_partition_param": (C.c_int, [_i64, _i64, _i64, _i64, _P(abi.BlockSpec), _i64, _P(_i64)]),
    "asg_blockset_create": (C.c_int, [C.c_int, _P(abi.OptimizerConfig), _P(abi.SchedulerConfig),
                                      _P(abi.ParamDesc), _i64, _i32, _i32, _i32, _u64, _P(_vp)]),
    "asg_blockset_destroy": (C.c_int, [_vp]),
    "asg_blockset_bind_params": (C.c_int, [_vp, _P(abi.ParamDesc), _i64]),
    "asg_blockset_num_blocks": (C.c_int, [_vp, _P(_i64)]),
    "asg_blockset_block_info": (C.c_int, [_vp, _i64, _P(abi.BlockInfo)]),
    "asg_blockset_state_bytes": (C.c_int, [_vp, _P(_u64)]),
    "asg_blockset_workspace_bytes": (C.c_int, [_vp, _P(_u64)]),
    "asg_store_config_defaults": (C.c_int, [_P(abi.StoreConfig)]),
    "asg_tierstore_create": (C.c_int, [_P(abi.StoreConfig), _P(_vp)]),
    "asg_tierstore_destroy": (C.c_int, [_vp]),
    "asg_tier_put": (C.c_int, [_vp, C.c_char_p, _i32, _vp, _u64, _i32, _P(abi.EntryView)]),
    "asg_tier_put_device": (C.c_int, [_vp, C.c_char_p, _i32, _vp, _u64, _i32, _P(abi.EntryView)]),
    "asg_tier_get": (C.c_int, [_vp, C.c_char_p, _i32, _vp, _u64, _P(_u64), _P(_i32)]),
    "asg_tier_device_ptr": (C.c_int, [_vp, C.c_char_p, _i32, _P(_vp)]),
    "asg_tier_demote": (C.c_int, [_vp, C.c_char_p, _i32, _i32]),
    "asg_tier_promote": (C.c_int, [_vp, C.c_char_p, _i32, _i32]),
    "asg_tier_reclaim": (C.c_int, [_vp, C.c_char_p, _i32, _P(_u64)]),
    "asg_tier_flush": (C.c_int, [_vp, C.c_char_p, _i32]),
    "asg_tier_pin": (C.c_int, [_vp, C.c_char_p, _i32]),
    "asg_tier_unpin": (C.c_int, [_vp, C.c_char_p, _i32]),
    "asg_tier_prefetch": (C.c_int, [_vp, C.c_char_p, _i32, _i32, _P(_u64)]),
    "asg_tier_drain_ready": (C.c_int, [_vp, _i32, _P(_i32)]),
    "asg_tier_advance_step": (C.c_int, [_vp, _i64]),
    "asg_tier_contains": (C.c_int, [_vp, C.c_char_p, _i32, _P(_i32)]),
    "asg_tier_inspect": (C.c_int, [_vp, C.c_char_p, _i32, _P(abi.EntryView)]),
    "asg_tier_gauges": (C.c_int, [_vp, _P(abi.Residency)]),
    "asg_tier_counters": (C.c_int, [_vp, _P(abi.IoCounters)]),
    "asg_tier_audit": (C.c_int, [_vp]),
    "asg_blockset_attach_store": (C.c_int, [_vp, _vp]),
    "asg_on_hook": (C.c_int, [_vp, _i32, _i64]),
    "asg_synth_gradients": (C.c_int, [_vp, _u64, _i64, _vp]),
    "asg_blockset_stream": (C.c_int, [_vp, _P(_vp)]),
    "asg_grad_sqnorm": (C.c_int, [_vp, _vp, _P(_f64), _P(_i32)]),
    "asg_accumulate": (C.c_int, [_vp, _f64, _vp]),
    "asg_maybe_dispatch": (C.c_int, [_vp, _i64, _P(_i64)]),
    "asg_staleness_barrier": (C.c_int, [_vp, _i64, _P(_f64)]),
    "asg_precondition_apply": (C.c_int, [_vp, _i64, _f64, _f64, _vp]),
    "asg_step_end": (C.c_int, [_vp, _i64]),
    "asg_step": (C.c_int, [_vp, _i64, _f64, _f64, _vp]),
    "asg_clock_advance": (C.c_int, [_vp, _f64]),
    "asg_get_freshness": (C.c_int, [_vp, _i64, _P(abi.Freshness)]),
    "asg_get_stats": (C.c_int, [_vp, _P(abi.PoolStats)]),
    "asg_get_events": (C.c_int, [_vp, _P(abi.Event), _i64, _P(_i64)]),
    "asg_synchronize": (C.c_int, [_vp]),
    "asg_block_read": (C.c_int, [_vp, _i64, _i32, _P(_f64), _i64]),
    "asg_block_write": (C.c_int, [_vp, _i64, _i32, _P(_f64), _i64]),
    "asg_block_set_counters": (C.c_int, [_vp, _i64, _u64, _i64, _i64]),
    "asg_block_accumulate_f64": (C.c_int, [_vp, _i64, _P(_f64), _i64]),
    "asg_block_refresh_f64": (C.c_int, [_vp, _i64, _i64]),
    "asg_block_precondition_f64": (C.c_int, [_vp, _i64, _P(_f64), _i64, _P(_f64)]),
    "asg_block_soap_step_f64": (C.c_int, [_vp, _i64, _P(_f64), _i64, _P(_f64)]),
    "asg_plan_owners": (C.c_int, [_P(abi.OptimizerConfig), _P(_i64), _P(_i64), _i64, _i32, _P(_i32), _i64, _P(_i64)]),
    "asg_shard_elems": (C.c_int, [_vp, _i32, _P(_i64)]),
    "asg_gather_stride": (C.c_int, [_vp, _P(_i64)]),
    "asg_pack_grads": (C.c_int, [_vp, _vp, _vp]),
    "asg_unpack_reduced_grads": (C.c_int, [_vp, _vp, _f32, _vp]),
    "asg_grad_sqnorm_owned": (C.c_int, [_vp, _vp, _P(_f64), _P(_i32)]),
    "asg_pack_owned": (C.c_int, [_vp, _vp, _vp]),
    "asg_unpack_gathered": (C.c_int, [_vp, _vp, _i64, _vp]),
    "asg_launch_count": (C.c_int, [_P(_u64)]),
    "asg_profile_enable": (C.c_int, [_vp, _i32]),
    "asg_get_kernel_stats": (C.c_int, [_vp, _P(abi.KernelStats), _i32]),
    "asg_gemm_tn": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _f32, _f32, _i32, _vp]),
    "asg_sym_eig_batched": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp]),
    "asg_sym_eig_batched_f32": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp]),
    "asg_set_allgather_buckets": (C.c_int, [_vp, _i32]),
    "asg_bucket_count": (C.c_int, [_vp, _P(_i64)]),
    "asg_bucket_stride": (C.c_int, [_vp, _i64, _P(_i64)]),
    "asg_bucket_pack": (C.c_int, [_vp, _i64, _vp, _vp]),
    "asg_bucket_unpack": (C.c_int, [_vp, _i64, _vp, _vp]),
    "asg_nccl_unique_id": (C.c_int, [_vp]),
    "asg_nccl_comm_init": (C.c_int, [_i32, _i32, _vp, _P(_vp)]),
    "asg_nccl_comm_destroy": (C.c_int, [_vp]),
    "asg_allgather_params": (C.c_int, [_vp, _vp, _vp]),
    "asg_set_allgather_comm": (C.c_int, [_vp, _vp, _i32]),
    "asg_snapshot_factors": (C.c_int, [_vp, _i64, _P(_vp)]),
    "asg_snapshot_checksum": (C.c_int, [_vp, _P(_u64)]),
    "asg_snapshot_destroy": (C.c_int, [_vp]),
    "asg_compute_refresh": (C.c_int, [_vp, _vp, _P(_vp)]),
    "asg_install_refresh": (C.c_int, [_vp, _i64, _vp, _i64]),
    "asg_refresh_result_destroy": (C.c_int, [_vp]),
    "asg_block_replicated_state": (C.c_int, [_vp, _i64, _P(_f64), _i64]),
    "asg_block_load_replicated_state": (C.c_int, [_vp, _i64, _P(_f64), _i64]),
    "asg_pack_spd_f32": (C.c_int, [_vp, _i64, _i64, _vp, _vp]),
    "asg_unpack_spd_f32": (C.c_int, [_vp, _i64, _i64, _vp, _vp]),
    "asg_adam_state_create": (C.c_int, [_i64, _i64, _P(_vp)]),
    "asg_adam_state_destroy": (C.c_int, [_vp]),
    "asg_adamw_step_f64": (C.c_int, [_vp, _P(_f64), _P(abi.OptimizerConfig), _P(_f64)]),
    "asg_apply_update_f64": (C.c_int, [_P(_f64), _P(_f64), _i64, _i64, _P(abi.OptimizerConfig), _f64]),
    "asg_get_hbm_stats": (C.c_int, [_vp, _P(abi.HbmStats), _i32]),
    "asg_inv_root_batched_f32": (C.c_int, [_vp, _vp, _i64, _i64, _i32, C.c_double, _i32, _vp]),
}

EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def check(rc):
    if rc != abi.ASG_OK:
        abi.raise_for(rc, lib.asg_last_error().decode(errors="replace"))


def device_supported(device=0):
    return bool(lib.asg_device_supported(device))


def optimizer_defaults(method):
    c = abi.OptimizerConfig()
    check(lib.asg_optimizer_defaults(method, C.byref(c)))
    return c


def validate(cfg):
    check(lib.asg_optimizer_validate(C.byref(cfg)))


def scheduler_defaults():
    s = abi.SchedulerConfig()
    check(lib.asg_scheduler_defaults(C.byref(s)))
    return s


def config_from_json(text):
    """(OptimizerConfig, SchedulerConfig, precision) from a RunConfig JSON string."""
    o, s, p = abi.OptimizerConfig(), abi.SchedulerConfig(), _i32()
    check(lib.asg_config_from_json(text.encode(), C.byref(o), C.byref(s), C.byref(p)))
    return o, s, p.value


def partition_param(rows, cols, limit, param_index=0):
    n = _i64()
    check(lib.asg_partition_param(param_index, rows, cols, limit, None, 0, C.byref(n)))
    out = (abi.BlockSpec * max(1, n.value))()
    check(lib.asg_partition_param(param_index, rows, cols, limit, out, n.value, C.byref(n)))
    return [out[i] for i in range(n.value)]


def plan_owners(opt, shapes, world):
    """Owner rank of every unit (block or 1-D AdamW parameter), LPT over `world`."""
    rows = (C.c_int64 * max(1, len(shapes)))(*[s[0] if len(s) > 1 else 1 for s in shapes])
    cols = (C.c_int64 * max(1, len(shapes)))(*[s[-1] if len(s) > 1 else s[0] for s in shapes])
    n = _i64()
    check(lib.asg_plan_owners(C.byref(opt), rows, cols, len(shapes), world, None, 0, C.byref(n)))
    out = (C.c_int32 * max(1, n.value))()
    check(lib.asg_plan_owners(C.byref(opt), rows, cols, len(shapes), world, out, n.value, C.byref(n)))
    return [out[i] for i in range(n.value)]
