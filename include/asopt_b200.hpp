// SPDX-License-Identifier: Apache-2.0
//
// asopt_b200.hpp — header-only C++ shim that re-exposes the reference's
// optimizer interface (proj/include/asopt/precond.hpp, errors.hpp) over the
// C-ABI of include/asteria_b200.h, so C++ callers written against
// `asopt::` port by changing the namespace to `asopt::b200::`.
//
//   reference                                  this shim
//   asopt::OptimizerConfig  precond.hpp:27-44  asopt::b200::OptimizerConfig (+ Method::KlShampoo)
//   asopt::partition_param  precond.hpp:59     asopt::b200::partition_param
//   asopt::PrecondBlock     precond.hpp:63-75  asopt::b200::PrecondBlock (state lives in HBM)
//   accumulate_factors      precond.hpp:105    accumulate_factors
//   refresh_inverse         precond.hpp:101    refresh_inverse (pure: returns a refreshed copy)
//   precondition_shampoo    precond.hpp:109    precondition_shampoo (also KL-Shampoo)
//   precondition_soap       precond.hpp:113    precondition_soap
//   soap_scaled_step        precond.hpp:119    soap_scaled_step
//   FactorSnapshot / snapshot_factors / compute_refresh / install_refresh
//                           precond.hpp:77-98  same names (state in HBM; compute is pure)
//   AdamState / adamw_step / apply_update
//                           precond.hpp:122-134 same names (the step fuses them on the device)
//   replicated_state / load_replicated_state
//                           precond.hpp:138-139 same names (flat std::vector<double>)
//   pack_spd / unpack_spd   densela.hpp:124-142 same names on host vectors (index shuffle only)
//   asopt::*Error           errors.hpp:10-47   asopt::b200::*Error, thrown from status codes
//
// Matrices cross the boundary as host row-major double (`Matd`, the
// reference's Eigen `Matd` is row-major double too, densela.hpp:29); inside,
// state is fp32 on the GPU (3xTF32 tensor-core products, see DESIGN.md §4 for
// the stated tolerances). In the optimizer step, `apply_update` / `adamw_step`
// are fused into the update GEMM's epilogue (asg_precondition_apply /
// asg_step); the per-call versions here run their own device kernels. The
// shim adds no CPU arithmetic.
//
// Link with -lasteria_b200 (paper_2605_16184_b200/csrc/build/).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "asteria_b200.h"

namespace asopt {
namespace b200 {

// ---- errors (errors.hpp:10-47) ---------------------------------------------
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NonFiniteError : Error { using Error::Error; };
struct NoConvergenceError : Error { using Error::Error; };
struct NotPsdError : Error { using Error::Error; };
struct LayoutMismatchError : Error { using Error::Error; };
struct ShapeMismatchError : Error { using Error::Error; };
struct StaleUninitializedError : Error { using Error::Error; };
struct MissingKeyError : Error { using Error::Error; };
struct WorkerPoolDownError : Error { using Error::Error; };
struct ConfigInvalidError : Error { using Error::Error; };
struct AuditError : Error { using Error::Error; };
struct CapacityExhaustedError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct PinnedEntryError : Error { using Error::Error; };
struct DirtyNotPersistedError : Error { using Error::Error; };
// GPU-layer failures (no reference counterpart)
struct DeviceError : Error { using Error::Error; };

inline void check(int rc) {
    if (rc == ASG_OK) return;
    const std::string msg = asg_last_error();
    switch (rc) {
        case ASG_ERR_NON_FINITE: throw NonFiniteError(msg);
        case ASG_ERR_NO_CONVERGENCE: throw NoConvergenceError(msg);
        case ASG_ERR_NOT_PSD: throw NotPsdError(msg);
        case ASG_ERR_LAYOUT_MISMATCH: throw LayoutMismatchError(msg);
        case ASG_ERR_SHAPE_MISMATCH: throw ShapeMismatchError(msg);
        case ASG_ERR_STALE_UNINITIALIZED: throw StaleUninitializedError(msg);
        case ASG_ERR_WORKER_POOL_DOWN: throw WorkerPoolDownError(msg);
        case ASG_ERR_CONFIG_INVALID: throw ConfigInvalidError(msg);
        case ASG_ERR_AUDIT: throw AuditError(msg);
        case ASG_ERR_MISSING_KEY: throw MissingKeyError(msg);
        case ASG_ERR_CAPACITY_EXHAUSTED: throw CapacityExhaustedError(msg);
        case ASG_ERR_IO: throw IoError(msg);
        case ASG_ERR_PINNED_ENTRY: throw PinnedEntryError(msg);
        case ASG_ERR_DIRTY_NOT_PERSISTED: throw DirtyNotPersistedError(msg);
        default: throw DeviceError(msg);
    }
}

// ---- dense host matrix (row-major double, like densela.hpp:29 Matd) ---------
struct Matd {
    int64_t rows = 0, cols = 0;
    std::vector<double> data;
    Matd() = default;
    Matd(int64_t r, int64_t c, double fill = 0.0) : rows(r), cols(c), data(size_t(r * c), fill) {}
    static Matd Zero(int64_t r, int64_t c) { return Matd(r, c); }
    static Matd Identity(int64_t r, int64_t c) {
        Matd m(r, c);
        for (int64_t i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
        return m;
    }
    double& operator()(int64_t i, int64_t j) { return data[size_t(i * cols + j)]; }
    double operator()(int64_t i, int64_t j) const { return data[size_t(i * cols + j)]; }
    const double* ptr() const { return data.data(); }
    double* ptr() { return data.data(); }
};

// ---- configuration (precond.hpp:19-44) ---------------------------------------
enum class Method { AdamW = ASG_METHOD_ADAMW, Shampoo = ASG_METHOD_SHAMPOO, Soap = ASG_METHOD_SOAP,
                    KlShampoo = ASG_METHOD_KL_SHAMPOO };
enum class Accumulation { Sum = ASG_ACCUM_SUM, Ema = ASG_ACCUM_EMA };

struct OptimizerConfig {
    Method method = Method::AdamW;
    double lr = 1e-3;
    double beta1 = 0.9;
    double beta2 = 0.95;
    double eps = 1e-8;
    double weight_decay = 0.0;
    int64_t precondition_frequency = 10;
    Accumulation accumulation = Accumulation::Sum;
    double damping = 1e-8;
    int64_t block_dim_limit = 2048;

    asg_optimizer_config to_c() const {
        asg_optimizer_config c{};
        c.method = int32_t(method);
        c.accumulation = int32_t(accumulation);
        c.lr = lr;
        c.beta1 = beta1;
        c.beta2 = beta2;
        c.eps = eps;
        c.weight_decay = weight_decay;
        c.precondition_frequency = precondition_frequency;
        c.damping = damping;
        c.block_dim_limit = block_dim_limit;
        return c;
    }
    static OptimizerConfig from_c(const asg_optimizer_config& c) {
        OptimizerConfig o;
        o.method = Method(c.method);
        o.accumulation = Accumulation(c.accumulation);
        o.lr = c.lr;
        o.beta1 = c.beta1;
        o.beta2 = c.beta2;
        o.eps = c.eps;
        o.weight_decay = c.weight_decay;
        o.precondition_frequency = c.precondition_frequency;
        o.damping = c.damping;
        o.block_dim_limit = c.block_dim_limit;
        return o;
    }
    void validate() const {  // precond.cpp:34-42
        const asg_optimizer_config c = to_c();
        check(asg_optimizer_validate(&c));
    }
    static OptimizerConfig defaults_for(Method m) {  // precond.cpp:44-62
        asg_optimizer_config c{};
        check(asg_optimizer_defaults(int32_t(m), &c));
        return from_c(c);
    }
};

// ---- blocking (precond.hpp:47-60) ----------------------------------------------
struct BlockSpec {
    std::string param_id;
    int64_t row_begin = 0, row_end = 0, col_begin = 0, col_end = 0, block_dim_limit = 0;
    int64_t rows() const { return row_end - row_begin; }
    int64_t cols() const { return col_end - col_begin; }
    std::string id() const {  // precond.cpp:64-67
        return param_id + "[" + std::to_string(row_begin) + ":" + std::to_string(row_end) + "," +
               std::to_string(col_begin) + ":" + std::to_string(col_end) + "]";
    }
};

inline std::vector<BlockSpec> partition_param(const std::string& param_id, int64_t rows, int64_t cols,
                                              int64_t limit) {
    int64_t n = 0;
    check(asg_partition_param(0, rows, cols, limit, nullptr, 0, &n));
    std::vector<asg_block_spec> raw(size_t(n > 0 ? n : 1));
    check(asg_partition_param(0, rows, cols, limit, raw.data(), n, &n));
    std::vector<BlockSpec> out;
    for (int64_t i = 0; i < n; ++i)
        out.push_back({param_id, raw[size_t(i)].row_begin, raw[size_t(i)].row_end, raw[size_t(i)].col_begin,
                       raw[size_t(i)].col_end, raw[size_t(i)].block_dim_limit});
    return out;
}

// ---- per-block state (precond.hpp:63-75), resident in HBM -----------------------
class PrecondBlock {
public:
    PrecondBlock(int64_t rows, int64_t cols, const OptimizerConfig& cfg, int32_t precision = ASG_PREC_3XTF32,
                 int device = 0)
        : rows_(rows), cols_(cols), cfg_(cfg), precision_(precision), device_(device) {
        open();
    }
    PrecondBlock(const PrecondBlock& o) : rows_(o.rows_), cols_(o.cols_), cfg_(o.cfg_), precision_(o.precision_),
                                          device_(o.device_) {
        open();
        copy_state_from(o);
    }
    PrecondBlock& operator=(PrecondBlock o) {
        std::swap(rows_, o.rows_);
        std::swap(cols_, o.cols_);
        std::swap(cfg_, o.cfg_);
        std::swap(precision_, o.precision_);
        std::swap(device_, o.device_);
        std::swap(h_, o.h_);
        return *this;
    }
    ~PrecondBlock() {
        if (h_) asg_blockset_destroy(h_);
    }

    int64_t rows() const { return rows_; }
    int64_t cols() const { return cols_; }
    Method method() const { return cfg_.method; }
    const OptimizerConfig& config() const { return cfg_; }
    asg_blockset* handle() const { return h_; }

    asg_block_info info() const {
        asg_block_info i{};
        check(asg_blockset_block_info(h_, 0, &i));
        return i;
    }
    uint64_t version() const { return info().version; }
    int64_t last_refresh_step() const { return info().last_refresh_step; }
    int64_t moment_steps() const { return info().moment_steps; }
    void set_counters(uint64_t version, int64_t last_refresh_step, int64_t moment_steps) {
        check(asg_block_set_counters(h_, 0, version, last_refresh_step, moment_steps));
    }

    Matd get(asg_role role) const {
        const int64_t r = (role == ASG_ROLE_FACTOR_L || role == ASG_ROLE_INV_L || role == ASG_ROLE_BASIS_L ||
                           role == ASG_ROLE_KL_INV_L)
                              ? rows_
                          : (role == ASG_ROLE_FACTOR_R || role == ASG_ROLE_INV_R || role == ASG_ROLE_BASIS_R ||
                             role == ASG_ROLE_KL_INV_R)
                              ? cols_
                          : (role == ASG_ROLE_EIGVALS_L || role == ASG_ROLE_EIGVALS_R) ? 1
                                                                                       : rows_;
        const int64_t c = (role == ASG_ROLE_FACTOR_L || role == ASG_ROLE_INV_L || role == ASG_ROLE_BASIS_L ||
                           role == ASG_ROLE_KL_INV_L || role == ASG_ROLE_EIGVALS_L)
                              ? rows_
                              : cols_;
        Matd m(r, c);
        check(asg_block_read(h_, 0, int32_t(role), m.ptr(), int64_t(m.data.size())));
        return m;
    }
    void set(asg_role role, const Matd& m) {
        check(asg_block_write(h_, 0, int32_t(role), m.ptr(), int64_t(m.data.size())));
    }
    Matd factor_l() const { return get(ASG_ROLE_FACTOR_L); }
    Matd factor_r() const { return get(ASG_ROLE_FACTOR_R); }
    Matd inv_l() const { return get(ASG_ROLE_INV_L); }
    Matd inv_r() const { return get(ASG_ROLE_INV_R); }
    Matd basis_l() const { return get(ASG_ROLE_BASIS_L); }
    Matd basis_r() const { return get(ASG_ROLE_BASIS_R); }
    Matd rotated_m() const { return get(ASG_ROLE_ROTATED_M); }
    Matd rotated_v() const { return get(ASG_ROLE_ROTATED_V); }

private:
    void open() {
        asg_optimizer_config c = cfg_.to_c();
        c.block_dim_limit = std::max<int64_t>(c.block_dim_limit, std::max(rows_, cols_));
        asg_scheduler_config s{};
        check(asg_scheduler_defaults(&s));
        s.pf = c.precondition_frequency;
        // Per-block entry points stage host data; no parameter/gradient binding.
        asg_param_desc p{nullptr, nullptr, rows_, cols_, cols_, cols_};
        check(asg_blockset_create(device_, &c, &s, &p, 1, precision_, 0, 1, 99, &h_));
    }
    void copy_state_from(const PrecondBlock& o) {
        static const asg_role soap_roles[] = {ASG_ROLE_FACTOR_L, ASG_ROLE_FACTOR_R, ASG_ROLE_BASIS_L,
                                              ASG_ROLE_BASIS_R, ASG_ROLE_ROTATED_M, ASG_ROLE_ROTATED_V,
                                              ASG_ROLE_EIGVALS_L, ASG_ROLE_EIGVALS_R};
        static const asg_role root_roles[] = {ASG_ROLE_FACTOR_L, ASG_ROLE_FACTOR_R, ASG_ROLE_INV_L, ASG_ROLE_INV_R};
        // (KL-Shampoo's inverses F^-1 = INV^2 are derived from the roots, not stored)
        if (cfg_.method == Method::Soap) {
            for (asg_role r : soap_roles) set(r, o.get(r));
        } else if (cfg_.method != Method::AdamW) {
            for (asg_role r : root_roles) set(r, o.get(r));
        }
        const asg_block_info i = o.info();
        set_counters(i.version, i.last_refresh_step, i.moment_steps);
    }

    int64_t rows_, cols_;
    OptimizerConfig cfg_;
    int32_t precision_;
    int device_;
    asg_blockset* h_ = nullptr;
};

inline void check_shape(const PrecondBlock& b, const Matd& g) {
    if (g.rows != b.rows() || g.cols != b.cols()) throw ShapeMismatchError("gradient shape does not match the block");
}

inline void check_cfg(const PrecondBlock& b, const OptimizerConfig& cfg) {
    const OptimizerConfig& o = b.config();
    if (cfg.method != o.method || cfg.accumulation != o.accumulation || cfg.beta1 != o.beta1 ||
        cfg.beta2 != o.beta2 || cfg.eps != o.eps || cfg.damping != o.damping)
        throw ConfigInvalidError("config differs from the one the block's GPU state was created with");
}

/// accumulate_factors (precond.cpp:173-189).
inline void accumulate_factors(PrecondBlock& b, const Matd& g, const OptimizerConfig& cfg) {
    check_shape(b, g);
    check_cfg(b, cfg);
    check(asg_block_accumulate_f64(b.handle(), 0, g.ptr(), g.cols));
}

/// refresh_inverse (precond.cpp:166-171): pure over `b`, returns the refreshed copy.
inline PrecondBlock refresh_inverse(const PrecondBlock& b, const OptimizerConfig& cfg, int64_t step) {
    check_cfg(b, cfg);
    PrecondBlock out(b);
    check(asg_block_refresh_f64(out.handle(), 0, step));
    return out;
}

/// The same, in place (avoids the state copy).
inline void refresh_inverse_inplace(PrecondBlock& b, const OptimizerConfig& cfg, int64_t step) {
    check_cfg(b, cfg);
    check(asg_block_refresh_f64(b.handle(), 0, step));
}

/// precondition_shampoo (precond.cpp:191-198); KL-Shampoo uses L^-1/2, R^-1/2.
inline Matd precondition_shampoo(const PrecondBlock& b, const Matd& g) {
    check_shape(b, g);
    Matd out(b.rows(), b.cols());
    check(asg_block_precondition_f64(b.handle(), 0, g.ptr(), g.cols, out.ptr()));
    return out;
}

/// soap_scaled_step (precond.cpp:208-223): updates the rotated moments.
inline Matd soap_scaled_step(PrecondBlock& b, const Matd& g, const OptimizerConfig& cfg) {
    check_shape(b, g);
    check_cfg(b, cfg);
    Matd out(b.rows(), b.cols());
    check(asg_block_soap_step_f64(b.handle(), 0, g.ptr(), g.cols, out.ptr()));
    return out;
}

/// precondition_soap (precond.cpp:200-206): StaleUninitialized before the first install.
inline Matd precondition_soap(PrecondBlock& b, const Matd& g, const OptimizerConfig& cfg) {
    if (b.version() == 0) throw StaleUninitializedError("precondition_soap: no refreshed basis installed");
    return soap_scaled_step(b, g, cfg);
}

// ---- the split refresh (precond.hpp:77-98) ---------------------------------------
/// FactorSnapshot: device copies of a block's L and R (snapshot_factors precond.cpp:112-117).
class FactorSnapshot {
public:
    FactorSnapshot(asg_blockset* bs, asg_snapshot* h) : bs_(bs), h_(h) {}
    FactorSnapshot(FactorSnapshot&& o) noexcept : bs_(o.bs_), h_(o.h_) { o.h_ = nullptr; }
    FactorSnapshot(const FactorSnapshot&) = delete;
    FactorSnapshot& operator=(const FactorSnapshot&) = delete;
    ~FactorSnapshot() {
        if (h_) asg_snapshot_destroy(h_);
    }
    /// snapshot_checksum (precond.cpp:114-115) over the fp32 factor bytes.
    uint64_t checksum() const {
        uint64_t c = 0;
        check(asg_snapshot_checksum(h_, &c));
        return c;
    }
    asg_blockset* blockset() const { return bs_; }
    const asg_snapshot* handle() const { return h_; }

private:
    asg_blockset* bs_;
    asg_snapshot* h_;
};

/// RefreshResult (precond.hpp:83-87), held in HBM until installed.
class RefreshResult {
public:
    explicit RefreshResult(asg_refresh_result* h) : h_(h) {}
    RefreshResult(RefreshResult&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    RefreshResult(const RefreshResult&) = delete;
    RefreshResult& operator=(const RefreshResult&) = delete;
    ~RefreshResult() {
        if (h_) asg_refresh_result_destroy(h_);
    }
    asg_refresh_result* release() {
        asg_refresh_result* h = h_;
        h_ = nullptr;
        return h;
    }

private:
    asg_refresh_result* h_;
};

inline FactorSnapshot snapshot_factors(const PrecondBlock& b) {
    asg_snapshot* h = nullptr;
    check(asg_snapshot_factors(b.handle(), 0, &h));
    return FactorSnapshot(b.handle(), h);
}

/// compute_refresh (precond.cpp:129-142): pure over the snapshot.
inline RefreshResult compute_refresh(const FactorSnapshot& snap, const OptimizerConfig& cfg) {
    (void)cfg;  // the snapshot's block carries the configuration its GPU state was created with
    asg_refresh_result* h = nullptr;
    check(asg_compute_refresh(snap.blockset(), snap.handle(), &h));
    return RefreshResult(h);
}

/// install_refresh (precond.cpp:144-164): consumes the result.
inline void install_refresh(PrecondBlock& b, RefreshResult&& r, int64_t step) {
    check(asg_install_refresh(b.handle(), 0, r.release(), step));
}

// ---- AdamW and apply (precond.hpp:122-134) ------------------------------------------
class AdamState {
public:
    AdamState(int64_t rows, int64_t cols) : rows_(rows), cols_(cols) { check(asg_adam_state_create(rows, cols, &h_)); }
    AdamState(AdamState&& o) noexcept : rows_(o.rows_), cols_(o.cols_), h_(o.h_) { o.h_ = nullptr; }
    AdamState(const AdamState&) = delete;
    AdamState& operator=(const AdamState&) = delete;
    ~AdamState() {
        if (h_) asg_adam_state_destroy(h_);
    }
    static AdamState zeros(int64_t rows, int64_t cols) { return AdamState(rows, cols); }
    int64_t rows() const { return rows_; }
    int64_t cols() const { return cols_; }
    asg_adam_state* handle() { return h_; }

private:
    int64_t rows_, cols_;
    asg_adam_state* h_ = nullptr;
};

/// adamw_step (precond.cpp:229-242): the bias-corrected Adam direction.
inline Matd adamw_step(AdamState& st, const Matd& g, const OptimizerConfig& cfg) {
    if (g.rows != st.rows() || g.cols != st.cols()) throw ShapeMismatchError("adamw_step: gradient shape mismatch");
    Matd out(g.rows, g.cols);
    const asg_optimizer_config c = cfg.to_c();
    check(asg_adamw_step_f64(st.handle(), g.ptr(), &c, out.ptr()));
    return out;
}

/// apply_update (precond.cpp:244-251): theta -= lr * lr_scale * (update + wd * theta).
inline void apply_update(Matd& theta, const Matd& update, const OptimizerConfig& cfg, double lr_scale = 1.0) {
    if (theta.rows != update.rows || theta.cols != update.cols) throw ShapeMismatchError("apply_update: shape mismatch");
    const asg_optimizer_config c = cfg.to_c();
    check(asg_apply_update_f64(theta.ptr(), update.ptr(), theta.rows, theta.cols, &c, lr_scale));
}

// ---- replicated state (precond.hpp:138-139) -----------------------------------------
inline std::vector<double> replicated_state(const PrecondBlock& b, Method /*method: the block's*/) {
    std::vector<double> flat(size_t(b.rows() * b.rows() + b.cols() * b.cols()));
    check(asg_block_replicated_state(b.handle(), 0, flat.data(), int64_t(flat.size())));
    return flat;
}
inline void load_replicated_state(PrecondBlock& b, Method /*method: the block's*/, const std::vector<double>& flat) {
    check(asg_block_load_replicated_state(b.handle(), 0, flat.data(), int64_t(flat.size())));
}

// ---- packed symmetric storage (densela.hpp:124-142) ---------------------------------
/// Lower triangle packed row-major: (0,0), (1,0), (1,1), (2,0), ...
inline std::vector<double> pack_spd(const Matd& m) {
    if (m.rows != m.cols) throw LayoutMismatchError("pack_spd: expected a square Full matrix");
    std::vector<double> p;
    p.reserve(size_t(m.rows * (m.rows + 1) / 2));
    for (int64_t i = 0; i < m.rows; ++i)
        for (int64_t j = 0; j <= i; ++j) p.push_back(m(i, j));
    return p;
}
inline Matd unpack_spd(const std::vector<double>& p, int64_t n) {
    if (int64_t(p.size()) != n * (n + 1) / 2) throw LayoutMismatchError("unpack_spd: expected PackedLower of size n(n+1)/2");
    Matd m(n, n);
    for (int64_t i = 0, k = 0; i < n; ++i)
        for (int64_t j = 0; j <= i; ++j, ++k) m(i, j) = m(j, i) = p[size_t(k)];
    return m;
}

// ---- tiered store (tierstore.hpp:71-114, tiers.hpp) ------------------------
enum class TierTag { Hot = ASG_TIER_HOT, Host = ASG_TIER_HOST, Cold = ASG_TIER_COLD };
enum class TensorRole : int32_t {
    FactorL = ASG_ROLE_FACTOR_L, FactorR = ASG_ROLE_FACTOR_R, InvFactorL = ASG_ROLE_INV_L,
    InvFactorR = ASG_ROLE_INV_R, BasisL = ASG_ROLE_BASIS_L, BasisR = ASG_ROLE_BASIS_R,
    RotatedM = ASG_ROLE_ROTATED_M, RotatedV = ASG_ROLE_ROTATED_V
};
struct TierKey {
    std::string block_id;
    TensorRole role;
};
struct StoreConfig {
    uint64_t hot_capacity_bytes = 1ull << 30;
    uint64_t host_capacity_bytes = 1ull << 30;
    std::string cold_path;
    double transfer_bandwidth_bytes_per_sec = 0.0;
    uint64_t transfer_latency_us = 0;
    int hot_device = -1;  // B200: the Hot tier's CUDA device (-1: host memory)
};
struct EntryView {
    TierTag tier = TierTag::Cold;
    uint64_t bytes = 0;
    bool dirty = false, pinned = false;
    int64_t last_touch_step = 0;
    bool staged_pending = false, staged_ready = false;
};

class TierStore {
  public:
    explicit TierStore(StoreConfig cfg) : cfg_(std::move(cfg)) {
        asg_store_config c;
        check(asg_store_config_defaults(&c));
        c.hot_capacity_bytes = cfg_.hot_capacity_bytes;
        c.host_capacity_bytes = cfg_.host_capacity_bytes;
        c.cold_path = cfg_.cold_path.c_str();
        c.transfer_bandwidth_bytes_per_sec = cfg_.transfer_bandwidth_bytes_per_sec;
        c.transfer_latency_us = cfg_.transfer_latency_us;
        c.hot_device = cfg_.hot_device;
        check(asg_tierstore_create(&c, &h_));
    }
    ~TierStore() {
        if (h_) asg_tierstore_destroy(h_);
    }
    TierStore(const TierStore&) = delete;
    TierStore& operator=(const TierStore&) = delete;

    EntryView put(const TierKey& k, const std::vector<std::byte>& bytes, TierTag tier) {
        asg_entry_view v;
        check(asg_tier_put(h_, k.block_id.c_str(), int32_t(k.role), bytes.data(), bytes.size(), int32_t(tier), &v));
        return view(v);
    }
    std::pair<std::vector<std::byte>, TierTag> get(const TierKey& k) {
        asg_entry_view v;
        check(asg_tier_inspect(h_, k.block_id.c_str(), int32_t(k.role), &v));
        std::vector<std::byte> out(v.bytes);
        uint64_t n = 0;
        int32_t t = 0;
        check(asg_tier_get(h_, k.block_id.c_str(), int32_t(k.role), out.data(), out.size(), &n, &t));
        return {std::move(out), TierTag(t)};
    }
    void demote(const TierKey& k, TierTag to) { check(asg_tier_demote(h_, k.block_id.c_str(), int32_t(k.role), int32_t(to))); }
    void promote(const TierKey& k, TierTag to) { check(asg_tier_promote(h_, k.block_id.c_str(), int32_t(k.role), int32_t(to))); }
    uint64_t reclaim(const TierKey& k) {
        uint64_t f = 0;
        check(asg_tier_reclaim(h_, k.block_id.c_str(), int32_t(k.role), &f));
        return f;
    }
    void flush(const TierKey& k) { check(asg_tier_flush(h_, k.block_id.c_str(), int32_t(k.role))); }
    void pin(const TierKey& k) { check(asg_tier_pin(h_, k.block_id.c_str(), int32_t(k.role))); }
    void unpin(const TierKey& k) { check(asg_tier_unpin(h_, k.block_id.c_str(), int32_t(k.role))); }
    uint64_t prefetch(const TierKey& k, TierTag to) {
        uint64_t t = 0;
        check(asg_tier_prefetch(h_, k.block_id.c_str(), int32_t(k.role), int32_t(to), &t));
        return t;
    }
    int drain_ready(int max_items) {
        int32_t n = 0;
        check(asg_tier_drain_ready(h_, max_items, &n));
        return n;
    }
    void advance_step(int64_t step) { check(asg_tier_advance_step(h_, step)); }
    bool contains(const TierKey& k) const {
        int32_t o = 0;
        check(asg_tier_contains(h_, k.block_id.c_str(), int32_t(k.role), &o));
        return o != 0;
    }
    EntryView inspect(const TierKey& k) const {
        asg_entry_view v;
        check(asg_tier_inspect(h_, k.block_id.c_str(), int32_t(k.role), &v));
        return view(v);
    }
    asg_residency gauges() const {
        asg_residency g;
        check(asg_tier_gauges(h_, &g));
        return g;
    }
    asg_io_counters counters() const {
        asg_io_counters c;
        check(asg_tier_counters(h_, &c));
        return c;
    }
    const StoreConfig& config() const { return cfg_; }
    void audit() const { check(asg_tier_audit(h_)); }
    asg_tierstore* handle() const { return h_; }

  private:
    static EntryView view(const asg_entry_view& v) {
        return EntryView{TierTag(v.tier), v.bytes, v.dirty != 0, v.pinned != 0, v.last_touch_step,
                         v.staged_pending != 0, v.staged_ready != 0};
    }
    StoreConfig cfg_;
    asg_tierstore* h_ = nullptr;
};

}  // namespace b200
}  // namespace asopt
