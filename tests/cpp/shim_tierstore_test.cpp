// SPDX-License-Identifier: Apache-2.0
// Reference tier-store test bodies (proj/tests/tierstore_test.cpp) through the
// C++ shim (include/asopt_b200.hpp) -- the call sites a reference C++ caller
// keeps. Hot tier in host memory (argv[2] = -1) or on a CUDA device.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "asopt_b200.hpp"

using namespace asopt::b200;

static int failed = 0, passed = 0;
#define CHECK(c)                                                           \
    do {                                                                   \
        if (c) {                                                           \
            ++passed;                                                      \
        } else {                                                           \
            ++failed;                                                      \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);     \
        }                                                                  \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
    }
    return false;
}

static std::vector<std::byte> payload(size_t n, unsigned fill) {  // tierstore_test.cpp:19-23
    std::vector<std::byte> v(n);
    for (size_t i = 0; i < n; ++i) v[i] = std::byte((fill + i) & 0xff);
    return v;
}
static TierKey key(const std::string& b, TensorRole r = TensorRole::InvFactorL) { return TierKey{b, r}; }

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";
    const int dev = argc > 2 ? std::atoi(argv[2]) : -1;
    auto cfg_for = [&](const char* name) {
        StoreConfig c;
        c.cold_path = dir + "/" + name;
        c.hot_device = dev;
        return c;
    };
    {  // put/get roundtrip per tier (:46-66)
        TierStore store(cfg_for("a.cold"));
        auto bytes = payload(1024, 1);
        store.put(key("b0"), bytes, TierTag::Hot);
        auto got = store.get(key("b0"));
        CHECK(got.first == bytes && got.second == TierTag::Hot);
        auto cold = payload(333, 9);
        store.put(key("b1"), cold, TierTag::Cold);
        CHECK(store.inspect(key("b1")).tier == TierTag::Cold);
        auto got2 = store.get(key("b1"));
        CHECK(got2.first == cold && got2.second == TierTag::Host);
        CHECK(store.counters().page_ins == 1);
        store.audit();
        CHECK(throws<MissingKeyError>([&] { store.get(key("nope")); }));
    }
    {  // capacity eviction (:76-96) and pinning (:98-113)
        StoreConfig c = cfg_for("e.cold");
        c.hot_capacity_bytes = 2048;
        TierStore store(c);
        store.put(key("a"), payload(1024, 1), TierTag::Hot);
        store.put(key("b"), payload(1024, 2), TierTag::Hot);
        store.get(key("a"));
        store.put(key("c"), payload(512, 3), TierTag::Hot);
        CHECK(store.inspect(key("b")).tier == TierTag::Host);
        CHECK(store.counters().evictions == 1);
        store.pin(key("a"));
        store.pin(key("c"));
        CHECK(throws<CapacityExhaustedError>([&] { store.put(key("d"), payload(1024, 4), TierTag::Hot); }));
        CHECK(throws<PinnedEntryError>([&] { store.demote(key("a"), TierTag::Host); }));
        CHECK(throws<DirtyNotPersistedError>([&] { store.reclaim(key("b")); }));
        store.audit();
    }
    {  // cold file layout is bit-exact (:169-191)
        StoreConfig c = cfg_for("fmt.cold");
        {
            TierStore store(c);
            store.put(key("fmt", TensorRole::InvFactorR), payload(64, 8), TierTag::Cold);
        }
        std::ifstream f(c.cold_path, std::ios::binary);
        std::vector<char> raw((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
        CHECK(raw.size() == 12 + 24 + 64);
        CHECK(std::memcmp(raw.data(), "ASTRCOLD", 8) == 0);
    }
    std::printf("%d passed, %d failed\n", passed, failed);
    return failed ? 1 : 0;
}
