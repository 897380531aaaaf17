# SPDX-License-Identifier: Apache-2.0
"""The reference's tier-store tests (proj/tests/tierstore_test.cpp) replayed
through the C-ABI store (asg_tierstore.cu, F3). Every case runs twice: with the
Hot tier in host memory (CPU, `-m "not gpu"`) and with the Hot tier in HBM on
cuda:0 (`-m gpu`), where Host is pinned memory and Host<->Hot moves are DMA
copies on the store's copy stream."""
import os
import random
import struct
import time

import pytest

from paper_2605_16184_b200 import abi

DEVICES = [pytest.param(-1, id="host-hot"), pytest.param(0, id="hbm-hot", marks=pytest.mark.gpu)]
HOT, HOST, COLD = abi.TIER_HOT, abi.TIER_HOST, abi.TIER_COLD


def payload(n, fill):  # tierstore_test.cpp:19-23
    return bytes(((fill + i) & 0xFF) for i in range(n))


def key(block, role=abi.INV_L):
    return (block, role)


def fnv1a64(data):  # bytes.hpp:14-22
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.fixture(params=DEVICES)
def mk(request, tmp_path):
    dev = request.param
    if dev >= 0:
        torch = pytest.importorskip("torch")
        if not torch.cuda.is_available():
            pytest.skip("no GPU")
    from paper_2605_16184_b200.tierstore import TierStore
    stores = []

    def make(name, **kw):
        s = TierStore(str(tmp_path / name), hot_device=dev, **kw)
        stores.append(s)
        return s

    make.dev = dev
    yield make
    for s in stores:
        s.close()


def test_put_get_roundtrip_per_tier(mk):  # :46-66
    store = mk("a.cold")
    b = payload(1024, 1)
    store.put(key("b0"), b, HOT)
    got, tier = store.get(key("b0"))
    assert got == b and tier == HOT
    cb = payload(333, 9)
    store.put(key("b1"), cb, COLD)
    assert store.inspect(key("b1")).tier == COLD
    got2, tier2 = store.get(key("b1"))
    assert got2 == cb
    assert tier2 == HOST  # promoted by the page-in
    assert store.counters().page_ins == 1
    store.audit()


def test_get_of_missing_key(mk):  # :68-74
    store = mk("m.cold")
    with pytest.raises(abi.MissingKeyError):
        store.get(key("nope"))


def test_capacity_eviction_demotes_the_coldest_unpinned_entry(mk):  # :76-96
    store = mk("e.cold", hot_capacity_bytes=2048, host_capacity_bytes=1 << 20)
    store.put(key("a"), payload(1024, 1), HOT)
    store.put(key("b"), payload(1024, 2), HOT)
    store.get(key("a"))  # b is now least recently touched
    store.put(key("c"), payload(512, 3), HOT)
    assert store.inspect(key("b")).tier == HOST
    assert store.inspect(key("a")).tier == HOT
    assert store.counters().evictions == 1
    g = store.gauges()
    assert g.hot_bytes == 1024 + 512 and g.host_bytes == 1024
    assert store.get(key("b"))[0] == payload(1024, 2)  # bytes survive the device -> host move
    store.audit()


def test_pinned_entries_block_eviction_and_demotion(mk):  # :98-113
    store = mk("p.cold", hot_capacity_bytes=1024)
    store.put(key("pinned"), payload(1024, 1), HOT)
    store.pin(key("pinned"))
    with pytest.raises(abi.CapacityExhaustedError):
        store.put(key("other"), payload(128, 2), HOT)
    with pytest.raises(abi.PinnedEntryError):
        store.demote(key("pinned"), HOST)
    store.unpin(key("pinned"))
    store.put(key("other"), payload(128, 2), HOT)
    assert store.inspect(key("pinned")).tier == HOST
    store.audit()


def test_demote_write_skip_for_clean_entries_write_for_dirty(mk):  # :115-134
    store = mk("d.cold")
    store.put(key("x"), payload(100, 4), HOST)
    assert store.inspect(key("x")).dirty
    store.flush(key("x"))
    assert not store.inspect(key("x")).dirty
    w = store.counters().file_writes
    store.demote(key("x"), COLD)
    assert store.counters().file_writes == w  # skipped
    assert store.counters().write_skips == 1
    store.put(key("y"), payload(100, 5), HOST)
    store.demote(key("y"), COLD)
    assert store.counters().file_writes == w + 1
    store.audit()


def test_reclaim_releases_bytes_and_preserves_content(mk):  # :136-153
    store = mk("r.cold")
    b = payload(777, 6)
    store.put(key("r"), b, HOST)
    with pytest.raises(abi.DirtyNotPersistedError):
        store.reclaim(key("r"))
    store.flush(key("r"))
    before = store.gauges().host_bytes
    assert store.reclaim(key("r")) == 777
    assert store.gauges().host_bytes == before - 777
    got, tier = store.get(key("r"))
    assert got == b and tier == HOST
    store.audit()


def test_promote_restores_exact_bytes_from_cold(mk):  # :155-167
    store = mk("pr.cold")
    b = payload(4096, 7)
    store.put(key("z"), b, COLD)
    store.promote(key("z"), HOT)
    got, tier = store.get(key("z"))
    assert got == b and tier == HOT
    store.audit()


def test_cold_file_layout_is_bit_exact(mk, tmp_path):  # :169-191
    store = mk("fmt.cold")
    b = payload(64, 8)
    store.put(key("fmt", abi.INV_R), b, COLD)
    raw = open(tmp_path / "fmt.cold", "rb").read()
    assert len(raw) == 12 + 24 + 64  # magic + u32 version + one record
    assert raw[:8] == b"ASTRCOLD"
    assert struct.unpack_from("<I", raw, 8)[0] == 1
    assert struct.unpack_from("<Q", raw, 12)[0] == fnv1a64(b"fmt/inv_r")
    assert struct.unpack_from("<Q", raw, 20)[0] == 64
    assert struct.unpack_from("<Q", raw, 28)[0] == fnv1a64(b)
    assert raw[36:] == b


def test_checksum_corruption_fails_loudly(mk, tmp_path):  # :193-206
    store = mk("bad.cold")
    store.put(key("c"), payload(128, 3), COLD)
    with open(tmp_path / "bad.cold", "r+b") as f:
        f.seek(12 + 24 + 17)
        f.write(b"\x5a")
    with pytest.raises(abi.IoError):
        store.get(key("c"))


def test_prefetch_is_asynchronous_coalesces_and_drains_without_blocking(mk):  # :208-232
    store = mk("pf.cold", transfer_latency_us=30000)  # 30 ms injected link delay
    store.put(key("pf"), payload(1 << 16, 2), COLD)
    t0 = time.perf_counter()
    t1 = store.prefetch(key("pf"), HOST)
    t2 = store.prefetch(key("pf"), HOST)
    assert time.perf_counter() - t0 < 0.015  # nowhere near the injected delay
    assert t1 == t2
    assert store.counters().transfers_coalesced == 1
    assert store.drain_ready(4) == 0  # not ready yet, must not block
    for _ in range(400):
        if store.drain_ready(4):
            break
        time.sleep(0.002)
    assert store.inspect(key("pf")).tier == HOST
    assert store.counters().transfers_started == 1
    store.audit()


def test_prefetch_to_hot_stages_off_the_caller(mk):
    """B200 mapping: a prefetch to Hot (cold read -> pinned -> HBM copy) is
    staged by the worker; drain installs it without another copy."""
    store = mk("ph.cold", transfer_latency_us=20000)
    b = payload(1 << 20, 5)
    store.put(key("w"), b, COLD)
    store.prefetch(key("w"), HOT)
    for _ in range(1000):
        if store.drain_ready(1):
            break
        time.sleep(0.002)
    v = store.inspect(key("w"))
    assert v.tier == HOT and not v.staged_pending and not v.staged_ready
    assert store.get(key("w")) == (b, HOT)
    if mk.dev >= 0:
        assert store.device_ptr(key("w"))  # resident in HBM
    assert store.counters().drains_installed == 1
    store.audit()


def test_drain_with_empty_queue_returns_zero(mk):  # :234-240
    store = mk("dq.cold")
    assert store.drain_ready(8) == 0


def test_enqueue_latency_independent_of_transfer_size(mk):  # :242-261
    store = mk("lat.cold", transfer_bandwidth_bytes_per_sec=1e6)  # 4 MiB ~= 4 s transfer
    store.put(key("small"), payload(1 << 10, 1), COLD)
    store.put(key("large"), bytes(4 << 20), COLD)
    for k in ("small", "large"):
        t0 = time.perf_counter()
        store.prefetch(key(k), HOST)
        assert time.perf_counter() - t0 < 0.010
    t0 = time.perf_counter()
    store.close()  # must not wait out the 4 s simulated transfer
    assert time.perf_counter() - t0 < 1.0


def test_stale_staged_copies_are_dropped_after_overwrite(mk):  # :263-279
    store = mk("st.cold")
    store.put(key("s"), payload(256, 1), COLD)
    store.prefetch(key("s"), HOST)
    for _ in range(400):
        if store.counters().transfers_completed:
            break
        time.sleep(0.001)
    fresh = payload(256, 9)
    store.put(key("s"), fresh, HOST)  # bumps the generation
    store.drain_ready(4)
    got, _ = store.get(key("s"))
    assert got == fresh
    assert store.counters().transfers_dropped >= 1
    store.audit()


def test_model_based_random_ops_against_an_in_memory_oracle(mk):  # :281-340
    store = mk("model.cold", hot_capacity_bytes=64 * 1024, host_capacity_bytes=128 * 1024)
    rng = random.Random(20240817)
    oracle = {}
    names = [f"blk{i}" for i in range(24)]
    tiers = (HOT, HOST, COLD)
    tolerated = (abi.MissingKeyError, abi.LayoutMismatchError, abi.PinnedEntryError,
                 abi.DirtyNotPersistedError, abi.CapacityExhaustedError)
    ops = 20000 if mk.dev < 0 else 8000
    checks = 0
    for op in range(ops):
        k = key(rng.choice(names))
        c = rng.randrange(100)
        try:
            if c < 30:
                b = payload(64 + rng.randrange(2048), rng.randrange(256))
                store.put(k, b, rng.choice(tiers))
                oracle[k[0]] = b
            elif c < 60:
                if k[0] in oracle:
                    got, _ = store.get(k)
                    assert got == oracle[k[0]]
                    checks += 1
                else:
                    with pytest.raises(abi.MissingKeyError):
                        store.get(k)
            elif c < 70:
                store.demote(k, rng.choice((HOST, COLD)))
            elif c < 78:
                store.promote(k, rng.choice((HOST, HOT)))
            elif c < 84:
                store.flush(k)
                store.reclaim(k)
            elif c < 92:
                store.prefetch(k, rng.choice((HOST, HOT)))
            else:
                store.drain_ready(rng.randrange(4))
        except tolerated:
            pass
        if op % 4096 == 0:
            store.audit()
        g = store.gauges()
        assert g.hot_bytes <= 64 * 1024 and g.host_bytes <= 128 * 1024
    for name, b in oracle.items():  # final sweep: every key byte-identical to the oracle
        assert store.get(key(name))[0] == b
    assert checks > 1000
    store.audit()


def test_config_requires_a_cold_path(tmp_path):
    from paper_2605_16184_b200.tierstore import TierStore
    with pytest.raises(abi.ConfigInvalidError):
        TierStore("")
