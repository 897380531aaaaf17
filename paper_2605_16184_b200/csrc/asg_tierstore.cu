// SPDX-License-Identifier: Apache-2.0
//
// Tiered store of optimizer state: the reference's
// TierStore (proj/include/asopt/tierstore.hpp, proj/src/tierstore.cpp) with
// its semantics kept -- residency gauges, least-recently-touched eviction one
// tier down, pinning, flush / reclaim, the append-only ASTRCOLD cold file,
// and prefetch by a transfer worker that drain_ready installs -- mapped onto
// the B200 memory hierarchy:
//
//   Hot  = device memory (HBM) of cfg.hot_device (stream-ordered allocations
//          on the store's copy stream), or host memory when hot_device = -1
//   Host = pinned host memory (DMA-able), or plain host memory without a GPU
//   Cold = the cold file, byte-identical to the reference's format
//
// Host <-> Hot moves are cudaMemcpyAsync on the store's own non-blocking copy
// stream. A prefetch is staged entirely by the worker thread (cold read ->
// pinned -> device), so the caller's enqueue cost is independent of the
// payload size and drain_ready installs a finished copy by moving a pointer.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <filesystem>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/asteria_b200.h"

namespace asg {
void set_last_error(const std::string& msg);  // asg_runtime.cu
}

namespace {

struct StoreFail {
    int code;
    std::string msg;
};

template <class F>
int store_guard(F&& f) {
    try {
        f();
        return ASG_OK;
    } catch (const StoreFail& e) {
        asg::set_last_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        asg::set_last_error("tierstore: host allocation failed");
        return ASG_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        asg::set_last_error(e.what());
        return ASG_ERR_INVALID_ARGUMENT;
    } catch (...) {
        asg::set_last_error("tierstore: unknown exception");
        return ASG_ERR_INVALID_ARGUMENT;
    }
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw StoreFail{e == cudaErrorMemoryAllocation ? ASG_ERR_OUT_OF_MEMORY : ASG_ERR_CUDA,
                        std::string("tierstore: ") + what + ": " + cudaGetErrorString(e)};
}

// FNV-1a 64 (bytes.hpp:14-22): key hashes and payload checksums of the cold file
uint64_t fnv1a64(const void* data, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= uint64_t(p[i]);
        h *= 0x100000001b3ull;
    }
    return h;
}

void put_u64_le(unsigned char* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
}
uint64_t get_u64_le(const unsigned char* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
    return v;
}

// TensorRole names (tiers.hpp:35-57) for the "block_id/role" key display;
// the KL-Shampoo / eigenvalue roles this library adds get their own names.
const char* role_name(int role) {
    static const char* names[] = {"factor_l", "factor_r", "inv_l",    "inv_r",    "basis_l",   "basis_r",
                                  "rotated_m", "rotated_v", "kl_inv_l", "kl_inv_r", "eigvals_l", "eigvals_r"};
    if (role < 0 || role > 11) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "tierstore: unknown role"};
    return names[role];
}

constexpr char kMagic[8] = {'A', 'S', 'T', 'R', 'C', 'O', 'L', 'D'};  // tierstore.cpp:14
constexpr uint32_t kRecordVersion = 1;
constexpr uint64_t kRecordHeaderBytes = 24;  // key hash + length + checksum

const char* tier_name(int t) { return t == ASG_TIER_HOT ? "Hot" : t == ASG_TIER_HOST ? "Host" : "Cold"; }
int tier_rank(int t) { return t == ASG_TIER_HOT ? 2 : t == ASG_TIER_HOST ? 1 : 0; }

// A resident payload: plain host, pinned host, or device memory.
struct Buf {
    enum Kind { NONE, VEC, PINNED, DEVICE };
    Kind kind = NONE;
    void* p = nullptr;
    uint64_t n = 0;
};

}  // namespace

struct asg_tierstore {
    asg_store_config cfg{};
    std::string cold_path;
    bool gpu = false;
    cudaStream_t copy = nullptr;

    struct Key {
        std::string id;
        int role;
        bool operator==(const Key& o) const { return role == o.role && id == o.id; }
        std::string display() const { return id + "/" + role_name(role); }
    };
    struct KeyHash {
        size_t operator()(const Key& k) const { return std::hash<std::string>{}(k.id) * 1000003u + size_t(k.role); }
    };
    struct Entry {
        Buf buffer;  // resident bytes (Hot / Host)
        int tier = ASG_TIER_COLD;
        uint64_t bytes = 0;
        bool dirty = false, pinned = false;
        int64_t last_touch_step = 0;
        uint64_t touch_seq = 0;
        uint64_t generation = 0;  // bumped on every content change
        bool in_flight = false;   // excluded from eviction while moving
        bool cold_valid = false;
        uint64_t cold_offset = 0, cold_length = 0, cold_checksum = 0;
    };
    struct Job {
        uint64_t ticket;
        Key key;
        int to;
        uint64_t bytes;
    };
    struct Staged {
        uint64_t ticket = 0;
        int to = ASG_TIER_HOST;
        Buf buf;
        uint64_t generation = 0;
    };
    struct InFlight {
        bool* f;
        explicit InFlight(bool* x) : f(x) { *f = true; }
        ~InFlight() { *f = false; }
    };

    std::mutex mu;
    std::unordered_map<Key, Entry, KeyHash> entries;
    asg_residency gauges{};
    asg_io_counters counters{};
    FILE* cold = nullptr;
    uint64_t cold_tail = 0;
    uint64_t touch_counter = 0;
    int64_t current_step = 0;
    uint64_t next_ticket = 1;
    std::deque<Job> jobs;
    std::unordered_map<Key, uint64_t, KeyHash> pending;
    std::unordered_map<Key, Staged, KeyHash> staged;
    std::deque<Key> ready;
    std::condition_variable cv;
    bool stop = false;
    std::thread worker;

    // ---- buffers --------------------------------------------------------
    void set_device() const {
        if (gpu) cuda_ok(cudaSetDevice(cfg.hot_device), "cudaSetDevice");
    }
    Buf::Kind kind_for(int tier) const {
        if (!gpu) return Buf::VEC;
        return tier == ASG_TIER_HOT ? Buf::DEVICE : Buf::PINNED;
    }
    Buf alloc(Buf::Kind k, uint64_t n) {
        Buf b;
        b.kind = k;
        b.n = n;
        if (k == Buf::VEC) {
            b.p = std::malloc(n ? n : 1);
            if (!b.p) throw std::bad_alloc();
        } else if (k == Buf::PINNED) {
            cuda_ok(cudaHostAlloc(&b.p, n ? n : 1, cudaHostAllocDefault), "cudaHostAlloc");
        } else {
            cuda_ok(cudaMallocAsync(&b.p, n ? n : 1, copy), "cudaMallocAsync");
        }
        return b;
    }
    void release(Buf& b) {
        if (b.kind == Buf::VEC) std::free(b.p);
        if (b.kind == Buf::PINNED) cudaFreeHost(b.p);
        if (b.kind == Buf::DEVICE) cudaFreeAsync(b.p, copy);
        b = Buf{};
    }
    // dst <- src (any kinds), complete on return
    void copy_into(Buf& dst, const void* src, Buf::Kind src_kind, uint64_t n) {
        if (dst.kind == Buf::DEVICE || src_kind == Buf::DEVICE) {
            cuda_ok(cudaMemcpyAsync(dst.p, src, n, cudaMemcpyDefault, copy), "cudaMemcpyAsync");
            cuda_ok(cudaStreamSynchronize(copy), "cudaStreamSynchronize");
        } else {
            std::memcpy(dst.p, src, n);
        }
    }
    Buf clone(const Buf& src, Buf::Kind k) {
        Buf b = alloc(k, src.n);
        copy_into(b, src.p, src.kind, src.n);
        return b;
    }
    // host-visible bytes of a buffer (device payloads are copied down)
    std::vector<unsigned char> host_bytes(const Buf& b) {
        std::vector<unsigned char> v(b.n);
        if (b.kind == Buf::DEVICE) {
            cuda_ok(cudaMemcpyAsync(v.data(), b.p, b.n, cudaMemcpyDeviceToHost, copy), "cudaMemcpyAsync");
            cuda_ok(cudaStreamSynchronize(copy), "cudaStreamSynchronize");
        } else if (b.n) {
            std::memcpy(v.data(), b.p, b.n);
        }
        return v;
    }

    uint64_t& gauge_of(int t) { return t == ASG_TIER_HOT ? gauges.hot_bytes : gauges.host_bytes; }
    void touch(Entry& e) {
        e.touch_seq = ++touch_counter;
        e.last_touch_step = current_step;
    }
    std::unordered_map<Key, Entry, KeyHash>::iterator find_or_throw(const Key& k) {
        auto it = entries.find(k);
        if (it == entries.end()) throw StoreFail{ASG_ERR_MISSING_KEY, "tierstore: missing key " + k.display()};
        return it;
    }
    asg_entry_view view_of(const Key& k, const Entry& e) const {
        asg_entry_view v{};
        v.tier = e.tier;
        v.bytes = e.bytes;
        v.dirty = e.dirty;
        v.pinned = e.pinned;
        v.last_touch_step = e.last_touch_step;
        v.staged_pending = pending.count(k) ? 1 : 0;
        v.staged_ready = staged.count(k) ? 1 : 0;
        return v;
    }

    // ---- cold file (tierstore.cpp:79-128) --------------------------------
    void write_cold_locked(const Key& k, Entry& e) {
        const std::vector<unsigned char> payload = host_bytes(e.buffer);
        unsigned char hdr[kRecordHeaderBytes];
        const std::string disp = k.display();
        put_u64_le(hdr, fnv1a64(disp.data(), disp.size()));
        put_u64_le(hdr + 8, payload.size());
        const uint64_t sum = fnv1a64(payload.data(), payload.size());
        put_u64_le(hdr + 16, sum);
        if (std::fseek(cold, long(cold_tail), SEEK_SET) != 0 || std::fwrite(hdr, 1, sizeof(hdr), cold) != sizeof(hdr) ||
            (!payload.empty() && std::fwrite(payload.data(), 1, payload.size(), cold) != payload.size()) ||
            std::fflush(cold) != 0)
            throw StoreFail{ASG_ERR_IO, "tierstore: cold write failed for " + disp};
        if (e.cold_valid) gauges.cold_bytes -= e.cold_length;
        e.cold_offset = cold_tail + kRecordHeaderBytes;
        e.cold_length = payload.size();
        e.cold_checksum = sum;
        e.cold_valid = true;
        cold_tail += kRecordHeaderBytes + payload.size();
        gauges.cold_bytes += e.cold_length;
        counters.file_writes += 1;
    }
    std::vector<unsigned char> read_cold_locked(const Key& k, const Entry& e) {
        const std::string disp = k.display();
        if (!e.cold_valid) throw StoreFail{ASG_ERR_IO, "tierstore: no cold copy for " + disp};
        std::vector<unsigned char> rec(kRecordHeaderBytes + e.cold_length);
        if (std::fseek(cold, long(e.cold_offset - kRecordHeaderBytes), SEEK_SET) != 0 ||
            std::fread(rec.data(), 1, rec.size(), cold) != rec.size())
            throw StoreFail{ASG_ERR_IO, "tierstore: cold read failed for " + disp};
        counters.file_reads += 1;
        if (get_u64_le(rec.data()) != fnv1a64(disp.data(), disp.size()) || get_u64_le(rec.data() + 8) != e.cold_length)
            throw StoreFail{ASG_ERR_IO, "tierstore: record header mismatch for " + disp};
        const uint64_t sum = get_u64_le(rec.data() + 16);
        std::vector<unsigned char> payload(rec.begin() + kRecordHeaderBytes, rec.end());
        if (fnv1a64(payload.data(), payload.size()) != sum || sum != e.cold_checksum)
            throw StoreFail{ASG_ERR_IO, "tierstore: checksum mismatch for " + disp};
        return payload;
    }
    Buf buf_from_host(const std::vector<unsigned char>& v, int tier) {
        Buf b = alloc(kind_for(tier), v.size());
        copy_into(b, v.data(), Buf::VEC, v.size());
        return b;
    }

    // ---- tier moves (tierstore.cpp:130-167) ---------------------------------
    void demote_locked(std::unordered_map<Key, Entry, KeyHash>::iterator it, int to, bool eviction) {
        Entry& e = it->second;
        if (e.pinned) throw StoreFail{ASG_ERR_PINNED_ENTRY, "tierstore: entry pinned: " + it->first.display()};
        if (tier_rank(to) >= tier_rank(e.tier))
            throw StoreFail{ASG_ERR_LAYOUT_MISMATCH, "tierstore: demote must move to a lower tier"};
        InFlight guard(&e.in_flight);
        if (to == ASG_TIER_COLD) {
            if (e.dirty) {
                write_cold_locked(it->first, e);
                e.dirty = false;
            } else {
                counters.write_skips += 1;
            }
            gauge_of(e.tier) -= e.bytes;
            release(e.buffer);
            e.tier = ASG_TIER_COLD;
        } else {  // Hot -> Host: make room below first; the bytes move device -> pinned
            ensure_capacity_locked(to, e.bytes);
            if (kind_for(to) != e.buffer.kind) {
                Buf nb = clone(e.buffer, kind_for(to));
                release(e.buffer);
                e.buffer = nb;
            }
            gauge_of(e.tier) -= e.bytes;
            e.tier = to;
            gauge_of(to) += e.bytes;
        }
        if (eviction) counters.evictions += 1;
    }
    void ensure_capacity_locked(int tier, uint64_t need) {
        if (tier == ASG_TIER_COLD) return;
        const uint64_t cap = tier == ASG_TIER_HOT ? cfg.hot_capacity_bytes : cfg.host_capacity_bytes;
        while (gauge_of(tier) + need > cap) {
            auto victim = entries.end();
            for (auto it = entries.begin(); it != entries.end(); ++it) {
                if (it->second.tier != tier || it->second.pinned || it->second.in_flight) continue;
                if (victim == entries.end() || it->second.touch_seq < victim->second.touch_seq) victim = it;
            }
            if (victim == entries.end())
                throw StoreFail{ASG_ERR_CAPACITY_EXHAUSTED,
                                std::string("tierstore: cannot make room in tier ") + tier_name(tier)};
            demote_locked(victim, tier == ASG_TIER_HOT ? ASG_TIER_HOST : ASG_TIER_COLD, true);
        }
    }

    // put (tierstore.cpp:169-211); src_kind says where `bytes` lives
    asg_entry_view put(const Key& k, const void* bytes, uint64_t n, int tier, Buf::Kind src_kind) {
        if (n == 0) throw StoreFail{ASG_ERR_SHAPE_MISMATCH, "tierstore: empty payload for " + k.display()};
        std::lock_guard<std::mutex> lk(mu);
        if (tier != ASG_TIER_COLD) {
            // room first, so a capacity failure leaves the old entry intact; the
            // replaced entry credits its own bytes and is shielded from eviction
            auto eit = entries.find(k);
            uint64_t credit = 0;
            if (eit != entries.end() && eit->second.tier == tier) credit = eit->second.bytes;
            if (eit != entries.end()) {
                InFlight guard(&eit->second.in_flight);
                ensure_capacity_locked(tier, n > credit ? n - credit : 0);
            } else {
                ensure_capacity_locked(tier, n);
            }
        }
        Entry& e = entries[k];
        InFlight guard(&e.in_flight);
        if (e.bytes > 0 && (e.tier == ASG_TIER_HOT || e.tier == ASG_TIER_HOST)) gauge_of(e.tier) -= e.bytes;
        if (e.cold_valid) {
            gauges.cold_bytes -= e.cold_length;  // the old record is orphaned
            e.cold_valid = false;
        }
        e.generation += 1;
        e.bytes = n;
        e.dirty = false;
        touch(e);
        release(e.buffer);
        if (tier == ASG_TIER_COLD) {
            e.buffer = alloc(Buf::VEC, n);
            copy_into(e.buffer, bytes, src_kind, n);
            write_cold_locked(k, e);
            release(e.buffer);
            e.tier = ASG_TIER_COLD;
        } else {
            e.buffer = alloc(kind_for(tier), n);
            copy_into(e.buffer, bytes, src_kind, n);
            e.tier = tier;
            e.dirty = true;
            gauge_of(tier) += n;
        }
        return view_of(k, e);
    }

    // ---- transfer worker (tierstore.cpp:310-366) --------------------------
    void transfer_worker() {
        if (gpu) cudaSetDevice(cfg.hot_device);
        std::unique_lock<std::mutex> lk(mu);
        while (true) {
            cv.wait(lk, [&] { return stop || !jobs.empty(); });
            if (stop) return;
            Job job = jobs.front();
            jobs.pop_front();
            counters.transfers_started += 1;
            // injected link delay outside the lock: the caller's enqueue cost is size-independent
            uint64_t delay_us = cfg.transfer_latency_us;
            if (cfg.transfer_bandwidth_bytes_per_sec > 0.0)
                delay_us += uint64_t(1e6 * double(job.bytes) / cfg.transfer_bandwidth_bytes_per_sec);
            if (delay_us > 0) {
                cv.wait_until(lk, std::chrono::system_clock::now() + std::chrono::microseconds(delay_us),
                              [&] { return stop; });
                if (stop) return;
            }
            auto it = entries.find(job.key);
            if (it == entries.end() || it->second.tier == job.to) {
                pending.erase(job.key);
                counters.transfers_dropped += 1;
                continue;
            }
            Entry& e = it->second;
            Staged s;
            s.ticket = job.ticket;
            s.to = job.to;
            s.generation = e.generation;
            try {
                if (e.tier == ASG_TIER_COLD) {
                    s.buf = buf_from_host(read_cold_locked(job.key, e), job.to);
                } else {
                    s.buf = clone(e.buffer, kind_for(job.to));  // e.g. pinned -> device DMA
                }
            } catch (const StoreFail&) {
                pending.erase(job.key);
                counters.transfers_dropped += 1;
                continue;  // surfaces on the next get
            }
            auto old = staged.find(job.key);
            if (old != staged.end()) release(old->second.buf);
            staged[job.key] = s;
            ready.push_back(job.key);
            counters.transfers_completed += 1;
        }
    }

    // install_staged (tierstore.cpp:368-402)
    void install_staged_locked(const Key& k, Staged&& s) {
        auto it = entries.find(k);
        pending.erase(k);
        if (it == entries.end()) {
            release(s.buf);
            counters.transfers_dropped += 1;
            return;
        }
        Entry& e = it->second;
        if (e.generation != s.generation || e.tier == s.to) {
            release(s.buf);
            counters.transfers_dropped += 1;
            return;
        }
        InFlight guard(&e.in_flight);
        try {
            if (s.to == ASG_TIER_COLD) {
                if (e.dirty) {
                    write_cold_locked(k, e);
                    e.dirty = false;
                }
                gauge_of(e.tier) -= e.bytes;
                release(e.buffer);
                release(s.buf);
                e.tier = ASG_TIER_COLD;
            } else {
                ensure_capacity_locked(s.to, s.buf.n);
                if (e.tier != ASG_TIER_COLD)
                    gauge_of(e.tier) -= e.bytes;
                else
                    e.dirty = false;
                release(e.buffer);
                e.buffer = s.buf;  // a pointer move: the copy was made by the worker
                s.buf = Buf{};
                e.tier = s.to;
                gauge_of(s.to) += e.bytes;
            }
            counters.drains_installed += 1;
        } catch (const StoreFail& f) {
            release(s.buf);
            if (f.code != ASG_ERR_CAPACITY_EXHAUSTED) throw;
            counters.transfers_dropped += 1;  // surfaces on the next get
        }
    }
};

extern "C" {

int asg_store_config_defaults(asg_store_config* out) {
    return store_guard([&] {
        if (!out) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        *out = asg_store_config{};
        out->hot_capacity_bytes = 1ull << 30;
        out->host_capacity_bytes = 1ull << 30;
        out->cold_path = nullptr;
        out->transfer_bandwidth_bytes_per_sec = 0.0;
        out->transfer_latency_us = 0;
        out->hot_device = -1;
    });
}

int asg_tierstore_create(const asg_store_config* cfg, asg_tierstore** out) {
    asg_tierstore* st = nullptr;
    const int rc = store_guard([&] {
        if (!cfg || !out) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        if (!cfg->cold_path || !*cfg->cold_path) throw StoreFail{ASG_ERR_CONFIG_INVALID, "tierstore: cold_path is empty"};
        st = new asg_tierstore();
        st->cfg = *cfg;
        st->cold_path = cfg->cold_path;
        st->cfg.cold_path = st->cold_path.c_str();
        st->gpu = cfg->hot_device >= 0;
        if (st->gpu) {
            cuda_ok(cudaSetDevice(cfg->hot_device), "cudaSetDevice");
            cuda_ok(cudaStreamCreateWithFlags(&st->copy, cudaStreamNonBlocking), "cudaStreamCreate");
        }
        const std::filesystem::path parent = std::filesystem::path(st->cold_path).parent_path();
        if (!parent.empty()) std::filesystem::create_directories(parent);
        st->cold = std::fopen(st->cold_path.c_str(), "w+b");  // truncate (tierstore.cpp:30-31)
        if (!st->cold) throw StoreFail{ASG_ERR_IO, "tierstore: cannot open cold file " + st->cold_path};
        unsigned char hdr[12];
        std::memcpy(hdr, kMagic, 8);
        for (int i = 0; i < 4; ++i) hdr[8 + i] = static_cast<unsigned char>((kRecordVersion >> (8 * i)) & 0xff);
        if (std::fwrite(hdr, 1, 12, st->cold) != 12 || std::fflush(st->cold) != 0)
            throw StoreFail{ASG_ERR_IO, "tierstore: cannot write the cold header"};
        st->cold_tail = 12;
        st->worker = std::thread([st] { st->transfer_worker(); });
        *out = st;
        st = nullptr;
    });
    if (st) {
        if (st->cold) std::fclose(st->cold);
        if (st->copy) cudaStreamDestroy(st->copy);
        delete st;
    }
    return rc;
}

int asg_tierstore_destroy(asg_tierstore* st) {
    return store_guard([&] {
        if (!st) return;
        {
            std::lock_guard<std::mutex> lk(st->mu);
            st->stop = true;
        }
        st->cv.notify_all();
        if (st->worker.joinable()) st->worker.join();  // never waits out an injected delay
        st->set_device();
        for (auto& kv : st->entries) st->release(kv.second.buffer);
        for (auto& kv : st->staged) st->release(kv.second.buf);
        if (st->copy) {
            cudaStreamSynchronize(st->copy);
            cudaStreamDestroy(st->copy);
        }
        if (st->cold) std::fclose(st->cold);
        delete st;
    });
}

#define ST_KEY                                                                             \
    if (!st || !block_id) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null argument"};     \
    role_name(role);                                                                       \
    st->set_device();                                                                      \
    const asg_tierstore::Key key{block_id, role};

static void check_tier(int t) {
    if (t != ASG_TIER_HOT && t != ASG_TIER_HOST && t != ASG_TIER_COLD)
        throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "tierstore: unknown tier"};
}

int asg_tier_put(asg_tierstore* st, const char* block_id, int32_t role, const void* bytes, uint64_t size, int32_t tier,
                 asg_entry_view* out) {
    return store_guard([&] {
        ST_KEY
        check_tier(tier);
        if (!bytes && size) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null payload"};
        const asg_entry_view v = st->put(key, bytes, size, tier, Buf::VEC);
        if (out) *out = v;
    });
}

int asg_tier_put_device(asg_tierstore* st, const char* block_id, int32_t role, const void* dev_bytes, uint64_t size,
                        int32_t tier, asg_entry_view* out) {
    return store_guard([&] {
        ST_KEY
        check_tier(tier);
        if (!st->gpu) throw StoreFail{ASG_ERR_UNSUPPORTED, "tierstore: no device tier (hot_device = -1)"};
        if (!dev_bytes && size) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null payload"};
        const asg_entry_view v = st->put(key, dev_bytes, size, tier, Buf::DEVICE);
        if (out) *out = v;
    });
}

int asg_tier_get(asg_tierstore* st, const char* block_id, int32_t role, void* out, uint64_t cap, uint64_t* size,
                 int32_t* tier) {
    return store_guard([&] {
        ST_KEY
        std::lock_guard<std::mutex> lk(st->mu);
        auto it = st->find_or_throw(key);
        asg_tierstore::Entry& e = it->second;
        if (size) *size = e.bytes;
        if (!out || cap < e.bytes) throw StoreFail{ASG_ERR_SHAPE_MISMATCH, "tierstore: output buffer too small"};
        st->touch(e);
        if (e.tier == ASG_TIER_COLD) {  // synchronous page-in promotes to Host (tierstore.cpp:218-226)
            std::vector<unsigned char> payload = st->read_cold_locked(key, e);
            st->ensure_capacity_locked(ASG_TIER_HOST, payload.size());
            st->release(e.buffer);
            e.buffer = st->buf_from_host(payload, ASG_TIER_HOST);
            e.tier = ASG_TIER_HOST;
            e.dirty = false;
            st->gauges.host_bytes += e.bytes;
            st->counters.page_ins += 1;
        }
        if (e.buffer.kind == Buf::DEVICE) {
            cuda_ok(cudaMemcpyAsync(out, e.buffer.p, e.bytes, cudaMemcpyDeviceToHost, st->copy), "cudaMemcpyAsync");
            cuda_ok(cudaStreamSynchronize(st->copy), "cudaStreamSynchronize");
        } else {
            std::memcpy(out, e.buffer.p, e.bytes);
        }
        if (tier) *tier = e.tier;
    });
}

int asg_tier_device_ptr(asg_tierstore* st, const char* block_id, int32_t role, void** dev_ptr) {
    return store_guard([&] {
        ST_KEY
        if (!dev_ptr) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        std::lock_guard<std::mutex> lk(st->mu);
        auto it = st->find_or_throw(key);
        if (it->second.tier != ASG_TIER_HOT || it->second.buffer.kind != Buf::DEVICE)
            throw StoreFail{ASG_ERR_LAYOUT_MISMATCH, "tierstore: entry is not resident in device memory"};
        // the payload's stream-ordered allocation is complete once the copy stream is
        cuda_ok(cudaStreamSynchronize(st->copy), "cudaStreamSynchronize");
        *dev_ptr = it->second.buffer.p;
    });
}

int asg_tier_demote(asg_tierstore* st, const char* block_id, int32_t role, int32_t to) {
    return store_guard([&] {
        ST_KEY
        check_tier(to);
        std::lock_guard<std::mutex> lk(st->mu);
        st->demote_locked(st->find_or_throw(key), to, false);
    });
}

int asg_tier_promote(asg_tierstore* st, const char* block_id, int32_t role, int32_t to) {
    return store_guard([&] {
        ST_KEY
        check_tier(to);
        std::lock_guard<std::mutex> lk(st->mu);
        auto it = st->find_or_throw(key);
        asg_tierstore::Entry& e = it->second;
        if (tier_rank(to) <= tier_rank(e.tier))
            throw StoreFail{ASG_ERR_LAYOUT_MISMATCH, "tierstore: promote must move to a higher tier"};
        asg_tierstore::InFlight guard(&e.in_flight);
        st->touch(e);
        if (e.tier == ASG_TIER_COLD) {
            std::vector<unsigned char> payload = st->read_cold_locked(key, e);
            st->ensure_capacity_locked(to, payload.size());
            st->release(e.buffer);
            e.buffer = st->buf_from_host(payload, to);
            e.dirty = false;
            st->gauge_of(to) += e.bytes;
        } else {
            st->ensure_capacity_locked(to, e.bytes);
            if (st->kind_for(to) != e.buffer.kind) {  // pinned -> device
                Buf nb = st->clone(e.buffer, st->kind_for(to));
                st->release(e.buffer);
                e.buffer = nb;
            }
            st->gauge_of(e.tier) -= e.bytes;
            st->gauge_of(to) += e.bytes;
        }
        e.tier = to;
    });
}

int asg_tier_reclaim(asg_tierstore* st, const char* block_id, int32_t role, uint64_t* freed) {
    return store_guard([&] {
        ST_KEY
        std::lock_guard<std::mutex> lk(st->mu);
        auto it = st->find_or_throw(key);
        asg_tierstore::Entry& e = it->second;
        uint64_t f = 0;
        if (e.tier != ASG_TIER_COLD) {
            if (e.dirty || !e.cold_valid)
                throw StoreFail{ASG_ERR_DIRTY_NOT_PERSISTED, "tierstore: reclaim of unpersisted entry " + key.display()};
            f = e.bytes;
            st->gauge_of(e.tier) -= f;
            st->release(e.buffer);
            e.tier = ASG_TIER_COLD;
        }
        if (freed) *freed = f;
    });
}

int asg_tier_flush(asg_tierstore* st, const char* block_id, int32_t role) {
    return store_guard([&] {
        ST_KEY
        std::lock_guard<std::mutex> lk(st->mu);
        auto it = st->find_or_throw(key);
        asg_tierstore::Entry& e = it->second;
        if (e.tier == ASG_TIER_COLD || !e.dirty) return;
        st->write_cold_locked(key, e);
        e.dirty = false;
    });
}

int asg_tier_pin(asg_tierstore* st, const char* block_id, int32_t role) {
    return store_guard([&] {
        ST_KEY
        std::lock_guard<std::mutex> lk(st->mu);
        st->find_or_throw(key)->second.pinned = true;
    });
}

int asg_tier_unpin(asg_tierstore* st, const char* block_id, int32_t role) {
    return store_guard([&] {
        ST_KEY
        std::lock_guard<std::mutex> lk(st->mu);
        st->find_or_throw(key)->second.pinned = false;
    });
}

int asg_tier_prefetch(asg_tierstore* st, const char* block_id, int32_t role, int32_t to, uint64_t* ticket) {
    return store_guard([&] {
        ST_KEY
        check_tier(to);
        uint64_t t = 0;
        {
            std::lock_guard<std::mutex> lk(st->mu);
            auto it = st->find_or_throw(key);
            st->counters.prefetch_requests += 1;
            auto pit = st->pending.find(key);
            if (pit != st->pending.end()) {
                st->counters.transfers_coalesced += 1;
                t = pit->second;
            } else {
                t = st->next_ticket++;
                st->pending.emplace(key, t);
                st->jobs.push_back(asg_tierstore::Job{t, key, to, it->second.bytes});
            }
        }
        st->cv.notify_one();
        if (ticket) *ticket = t;
    });
}

int asg_tier_drain_ready(asg_tierstore* st, int32_t max_items, int32_t* installed) {
    return store_guard([&] {
        if (!st) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        st->set_device();
        std::lock_guard<std::mutex> lk(st->mu);
        int n = 0;
        while (n < max_items && !st->ready.empty()) {
            const asg_tierstore::Key k = st->ready.front();
            st->ready.pop_front();
            auto sit = st->staged.find(k);
            if (sit == st->staged.end()) continue;
            asg_tierstore::Staged s = sit->second;
            st->staged.erase(sit);
            const uint64_t drops = st->counters.transfers_dropped;
            st->install_staged_locked(k, std::move(s));
            if (st->counters.transfers_dropped == drops) n += 1;
        }
        if (installed) *installed = n;
    });
}

int asg_tier_advance_step(asg_tierstore* st, int64_t step) {
    return store_guard([&] {
        if (!st) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        std::lock_guard<std::mutex> lk(st->mu);
        st->current_step = step;
    });
}

int asg_tier_contains(asg_tierstore* st, const char* block_id, int32_t role, int32_t* out) {
    return store_guard([&] {
        ST_KEY
        std::lock_guard<std::mutex> lk(st->mu);
        if (out) *out = st->entries.count(key) ? 1 : 0;
    });
}

int asg_tier_inspect(asg_tierstore* st, const char* block_id, int32_t role, asg_entry_view* out) {
    return store_guard([&] {
        ST_KEY
        std::lock_guard<std::mutex> lk(st->mu);
        auto it = st->find_or_throw(key);
        if (out) *out = st->view_of(key, it->second);
    });
}

int asg_tier_gauges(asg_tierstore* st, asg_residency* out) {
    return store_guard([&] {
        if (!st || !out) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        std::lock_guard<std::mutex> lk(st->mu);
        *out = st->gauges;
    });
}

int asg_tier_counters(asg_tierstore* st, asg_io_counters* out) {
    return store_guard([&] {
        if (!st || !out) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        std::lock_guard<std::mutex> lk(st->mu);
        *out = st->counters;
    });
}

int asg_tier_audit(asg_tierstore* st) {
    return store_guard([&] {
        if (!st) throw StoreFail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        std::lock_guard<std::mutex> lk(st->mu);
        uint64_t hot = 0, host = 0, cold = 0;
        for (const auto& kv : st->entries) {
            const asg_tierstore::Entry& e = kv.second;
            if (e.tier == ASG_TIER_HOT) hot += e.bytes;
            if (e.tier == ASG_TIER_HOST) host += e.bytes;
            if (e.cold_valid) cold += e.cold_length;
            if (e.tier != ASG_TIER_COLD && e.buffer.n != e.bytes)
                throw StoreFail{ASG_ERR_AUDIT, "tierstore: buffer size mismatch for " + kv.first.display()};
            if (e.tier == ASG_TIER_HOT && st->gpu && e.buffer.kind != Buf::DEVICE)
                throw StoreFail{ASG_ERR_AUDIT, "tierstore: Hot entry not in device memory: " + kv.first.display()};
            if (e.tier == ASG_TIER_COLD && e.dirty)
                throw StoreFail{ASG_ERR_AUDIT, "tierstore: dirty entry resident in Cold: " + kv.first.display()};
        }
        if (hot != st->gauges.hot_bytes || host != st->gauges.host_bytes || cold != st->gauges.cold_bytes)
            throw StoreFail{ASG_ERR_AUDIT, "tierstore: residency gauges out of sync"};
        if (hot > st->cfg.hot_capacity_bytes || host > st->cfg.host_capacity_bytes)
            throw StoreFail{ASG_ERR_AUDIT, "tierstore: capacity exceeded"};
    });
}

}  // extern "C"
