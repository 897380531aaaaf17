# SPDX-License-Identifier: Apache-2.0
"""Python mirror of the reference's ``asopt::TierStore`` (proj/include/asopt/
tierstore.hpp:71-114) over the C-ABI (``asg_tier_*``, asg_tierstore.cu).

Same method names, argument meaning and error classes as the reference:
keys are ``(block_id, role)`` (``TierKey`` tiers.hpp:45-51, role = an
``abi`` role such as ``abi.INV_L``), tiers are ``abi.TIER_HOT/HOST/COLD``,
payloads are ``bytes``. On a GPU box the Hot tier is HBM (``hot_device``);
``hot_device=-1`` keeps it in host memory.
"""
import ctypes as C

from . import abi
from .runtime import check, lib


def _key(k):
    block_id, role = k
    return block_id.encode(), int(role)


class TierStore:
    """TierStore (tierstore.hpp:71): put/get/demote/promote/reclaim/flush/pin/
    unpin/prefetch/drain_ready/advance_step/contains/inspect/gauges/counters/
    audit."""

    def __init__(self, cold_path, hot_capacity_bytes=1 << 30, host_capacity_bytes=1 << 30,
                 transfer_bandwidth_bytes_per_sec=0.0, transfer_latency_us=0, hot_device=-1):
        cfg = abi.StoreConfig()
        check(lib.asg_store_config_defaults(C.byref(cfg)))
        self._path = cold_path.encode()
        cfg.cold_path = self._path
        cfg.hot_capacity_bytes = hot_capacity_bytes
        cfg.host_capacity_bytes = host_capacity_bytes
        cfg.transfer_bandwidth_bytes_per_sec = transfer_bandwidth_bytes_per_sec
        cfg.transfer_latency_us = transfer_latency_us
        cfg.hot_device = hot_device
        self.config = cfg
        self._h = C.c_void_p()
        check(lib.asg_tierstore_create(C.byref(cfg), C.byref(self._h)))

    def close(self):
        if self._h:
            check(lib.asg_tierstore_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def put(self, key, payload, tier):
        b, r = _key(key)
        v = abi.EntryView()
        buf = C.create_string_buffer(bytes(payload), len(payload))
        check(lib.asg_tier_put(self._h, b, r, buf, len(payload), tier, C.byref(v)))
        return v

    def put_device(self, key, dev_ptr, size, tier):
        """put from device memory (a torch CUDA tensor's data_ptr())."""
        b, r = _key(key)
        v = abi.EntryView()
        check(lib.asg_tier_put_device(self._h, b, r, C.c_void_p(dev_ptr), size, tier, C.byref(v)))
        return v

    def get(self, key):
        """Returns (payload bytes, tier); a Cold entry is paged in to Host."""
        b, r = _key(key)
        size = C.c_uint64()
        tier = C.c_int32()
        rc = lib.asg_tier_get(self._h, b, r, None, 0, C.byref(size), C.byref(tier))
        if rc != abi.ShapeMismatchError.code:
            check(rc)
        out = C.create_string_buffer(max(1, size.value))
        check(lib.asg_tier_get(self._h, b, r, out, size.value, C.byref(size), C.byref(tier)))
        return out.raw[:size.value], tier.value

    def device_ptr(self, key):
        b, r = _key(key)
        p = C.c_void_p()
        check(lib.asg_tier_device_ptr(self._h, b, r, C.byref(p)))
        return p.value

    def demote(self, key, to):
        check(lib.asg_tier_demote(self._h, *_key(key), to))

    def promote(self, key, to):
        check(lib.asg_tier_promote(self._h, *_key(key), to))

    def reclaim(self, key):
        f = C.c_uint64()
        check(lib.asg_tier_reclaim(self._h, *_key(key), C.byref(f)))
        return f.value

    def flush(self, key):
        check(lib.asg_tier_flush(self._h, *_key(key)))

    def pin(self, key):
        check(lib.asg_tier_pin(self._h, *_key(key)))

    def unpin(self, key):
        check(lib.asg_tier_unpin(self._h, *_key(key)))

    def prefetch(self, key, to):
        t = C.c_uint64()
        check(lib.asg_tier_prefetch(self._h, *_key(key), to, C.byref(t)))
        return t.value

    def drain_ready(self, max_items):
        n = C.c_int32()
        check(lib.asg_tier_drain_ready(self._h, max_items, C.byref(n)))
        return n.value

    def advance_step(self, step):
        check(lib.asg_tier_advance_step(self._h, step))

    def contains(self, key):
        o = C.c_int32()
        check(lib.asg_tier_contains(self._h, *_key(key), C.byref(o)))
        return bool(o.value)

    def inspect(self, key):
        v = abi.EntryView()
        check(lib.asg_tier_inspect(self._h, *_key(key), C.byref(v)))
        return v

    def gauges(self):
        g = abi.Residency()
        check(lib.asg_tier_gauges(self._h, C.byref(g)))
        return g

    def counters(self):
        c = abi.IoCounters()
        check(lib.asg_tier_counters(self._h, C.byref(c)))
        return c

    def audit(self):
        check(lib.asg_tier_audit(self._h))
