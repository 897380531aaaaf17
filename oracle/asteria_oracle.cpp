// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY — the CPU oracle. Nothing in the product path
// (paper_2605_16184_b200/) may import, link or call this file; only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// use it, and only as the checker or the timed CPU baseline.
//
// A faithful fp64 restatement (no Eigen) of the reference's optimizer hot path:
//   densela  proj/include/asopt/densela.hpp:124-282
//   precond  proj/src/precond.cpp:11-279
//   schedule proj/src/asyncsched.cpp:108-221,268-286 (ShadowScheduler rules)
//   inputs   proj/tests/support/test_util.hpp:10-37 (mt19937_64 + libstdc++
//            std::normal_distribution, so inputs are bit-identical to the
//            reference tests' inputs on this toolchain)
// plus KL-Shampoo, which the reference leaves as a plug-in point:
//   L <- b L + (1-b)/n * G R^-1 G^T,  R <- b R + (1-b)/m * G^T L^-1 G,
//   update L^-1/2 G R^-1/2, inverses from the last (pf-refreshed) eigh.
//   (Lin et al. 2025, arXiv 2509.03378; parity for this part is unpinned by
//   the reference.)
//
// The reference itself cannot be compiled here (needs Eigen3, absent; see
// DESIGN.md "Oracle"), so the oracle is pinned by the reference's own
// known-answer tests (tests/test_oracle_*.py) and cross-checked with LAPACK.
//
// Matrix products use the plain i-k-j loop order; Eigen's blocked GEMM sums in
// a different order, so agreement with Eigen-built binaries is to rounding,
// not bitwise. Everything else (Jacobi rotation order, closed forms, sort,
// damping, EMA arithmetic) follows the reference operation by operation.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../include/asteria_b200.h"

namespace orc {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local std::string g_last_error;

template <class S>
struct Mat {
    int64_t r = 0, c = 0;
    std::vector<S> d;
    Mat() = default;
    Mat(int64_t rows, int64_t cols) : r(rows), c(cols), d(static_cast<size_t>(rows * cols), S(0)) {}
    S& operator()(int64_t i, int64_t j) { return d[static_cast<size_t>(i * c + j)]; }
    const S& operator()(int64_t i, int64_t j) const { return d[static_cast<size_t>(i * c + j)]; }
    static Mat identity(int64_t n) {
        Mat m(n, n);
        for (int64_t i = 0; i < n; ++i) m(i, i) = S(1);
        return m;
    }
    Mat transpose() const {
        Mat t(c, r);
        for (int64_t i = 0; i < r; ++i)
            for (int64_t j = 0; j < c; ++j) t(j, i) = (*this)(i, j);
        return t;
    }
    bool all_finite() const {
        for (const S& x : d)
            if (!std::isfinite(static_cast<double>(x))) return false;
        return true;
    }
};
using Matd = Mat<double>;

template <class S>
Mat<S> matmul(const Mat<S>& a, const Mat<S>& b) {  // densela.hpp:144-149
    if (a.c != b.r) throw Error(ASG_ERR_SHAPE_MISMATCH, "matmul: inner dimensions disagree");
    Mat<S> out(a.r, b.c);
    for (int64_t i = 0; i < a.r; ++i)
        for (int64_t k = 0; k < a.c; ++k) {
            const S aik = a(i, k);
            const S* brow = &b.d[static_cast<size_t>(k * b.c)];
            S* orow = &out.d[static_cast<size_t>(i * b.c)];
            for (int64_t j = 0; j < b.c; ++j) orow[j] += aik * brow[j];
        }
    return out;
}

template <class S>
Mat<S> symmetrized(const Mat<S>& m) {  // densela.hpp:152-156
    Mat<S> s(m.r, m.c);
    for (int64_t i = 0; i < m.r; ++i)
        for (int64_t j = 0; j < m.c; ++j) s(i, j) = (m(i, j) + m(j, i)) / S(2);
    return s;
}

template <class S>
Mat<S> gram_left(const Mat<S>& g) {  // densela.hpp:160-166
    if (!g.all_finite()) throw Error(ASG_ERR_NON_FINITE, "gram_left: non-finite input");
    return symmetrized(matmul(g, g.transpose()));
}

template <class S>
Mat<S> gram_right(const Mat<S>& g) {  // densela.hpp:169-175
    if (!g.all_finite()) throw Error(ASG_ERR_NON_FINITE, "gram_right: non-finite input");
    return symmetrized(matmul(g.transpose(), g));
}

template <class S>
struct EigenPair {  // densela.hpp:113-122
    std::vector<S> values;
    Mat<S> vectors;
    static EigenPair identity(int64_t n) {
        return {std::vector<S>(static_cast<size_t>(n), S(1)), Mat<S>::identity(n)};
    }
};

// Cyclic Jacobi, densela.hpp:182-264: <=30 sweeps, tol 1e-12*||A||_F, rotations
// in (p<q) order with the closed-form plane update, ascending stable sort.
template <class S>
EigenPair<S> sym_eig(const Mat<S>& m) {
    const int64_t n = m.r;
    if (m.r != m.c) throw Error(ASG_ERR_SHAPE_MISMATCH, "sym_eig: matrix is not square");
    Mat<S> a = m;
    if (!a.all_finite()) throw Error(ASG_ERR_NON_FINITE, "sym_eig: non-finite input");
    if (n == 0) return {};
    Mat<S> vt = Mat<S>::identity(n);
    S fro = 0;
    for (const S& x : a.d) fro += x * x;
    fro = std::sqrt(fro);
    const S tol = S(1e-12) * fro;
    constexpr int kMaxSweeps = 30;
    auto off_diag_norm = [&]() {
        S acc = 0;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = i + 1; j < n; ++j) acc += a(i, j) * a(i, j);
        return std::sqrt(S(2) * acc);
    };
    bool converged = (n == 1) || off_diag_norm() <= tol;
    for (int sweep = 0; sweep < kMaxSweeps && !converged; ++sweep) {
        for (int64_t p = 0; p < n - 1; ++p) {
            for (int64_t q = p + 1; q < n; ++q) {
                const S apq = a(p, q);
                if (apq == S(0)) continue;
                const S app = a(p, p);
                const S aqq = a(q, q);
                const S tau = (aqq - app) / (S(2) * apq);
                const S t = (tau >= S(0)) ? S(1) / (tau + std::sqrt(S(1) + tau * tau))
                                          : S(-1) / (-tau + std::sqrt(S(1) + tau * tau));
                const S c = S(1) / std::sqrt(S(1) + t * t);
                const S s = t * c;
                S* rp = &a.d[static_cast<size_t>(p * n)];
                S* rq = &a.d[static_cast<size_t>(q * n)];
                for (int64_t i = 0; i < n; ++i) {
                    const S x = rp[i];
                    const S y = rq[i];
                    rp[i] = c * x - s * y;
                    rq[i] = s * x + c * y;
                }
                rp[p] = app - t * apq;
                rq[q] = aqq + t * apq;
                rp[q] = S(0);
                rq[p] = S(0);
                for (int64_t i = 0; i < n; ++i) {
                    a(i, p) = rp[i];
                    a(i, q) = rq[i];
                }
                S* vp = &vt.d[static_cast<size_t>(p * n)];
                S* vq = &vt.d[static_cast<size_t>(q * n)];
                for (int64_t i = 0; i < n; ++i) {
                    const S x = vp[i];
                    const S y = vq[i];
                    vp[i] = c * x - s * y;
                    vq[i] = s * x + c * y;
                }
            }
        }
        converged = off_diag_norm() <= tol;
    }
    if (!converged) throw Error(ASG_ERR_NO_CONVERGENCE, "sym_eig: Jacobi sweep budget exhausted");
    std::vector<int64_t> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), int64_t(0));
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t i, int64_t j) { return a(i, i) < a(j, j); });
    EigenPair<S> out;
    out.values.resize(static_cast<size_t>(n));
    out.vectors = Mat<S>(n, n);
    for (int64_t k = 0; k < n; ++k) {
        out.values[static_cast<size_t>(k)] = a(order[k], order[k]);
        for (int64_t i = 0; i < n; ++i) out.vectors(i, k) = vt(order[k], i);
    }
    return out;
}

// Reconstruction V diag(w) V^T then symmetrize (densela.hpp:280-281).
template <class S>
Mat<S> reconstruct(const EigenPair<S>& eig, const std::vector<S>& w) {
    const int64_t n = eig.vectors.r;
    Mat<S> vw(n, n);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) vw(i, j) = eig.vectors(i, j) * w[static_cast<size_t>(j)];
    return symmetrized(matmul(vw, eig.vectors.transpose()));
}

// (m + damping I)^(-1/root_order), densela.hpp:267-282.
template <class S>
Mat<S> inv_root(const Mat<S>& m, int root_order, S damping) {
    if (root_order < 1) throw Error(ASG_ERR_SHAPE_MISMATCH, "inv_root: root_order must be >= 1");
    if (damping < S(0)) throw Error(ASG_ERR_NOT_PSD, "inv_root: negative damping");
    EigenPair<S> eig = sym_eig(m);
    const int64_t n = m.r;
    std::vector<S> w(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        const S damped = eig.values[static_cast<size_t>(i)] + damping;
        if (damped <= S(0))
            throw Error(ASG_ERR_NOT_PSD,
                        "inv_root: damped eigenvalue <= 0 at index " + std::to_string(i));
        w[static_cast<size_t>(i)] = std::pow(damped, S(-1) / S(root_order));
    }
    return reconstruct(eig, w);
}

// ---- inputs: test_util.hpp:10-26 ------------------------------------------
Matd random_matrix(int64_t rows, int64_t cols, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> dist(0.0, 1.0);
    Matd m(rows, cols);
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) m(i, j) = dist(rng);
    return m;
}

Matd random_spd(int64_t dim, uint64_t seed, double ridge) {
    Matd a = random_matrix(dim, dim, seed);
    Matd m = matmul(a, a.transpose());
    for (double& x : m.d) x /= static_cast<double>(dim);
    for (int64_t i = 0; i < dim; ++i) m(i, i) += ridge;
    return symmetrized(m);
}

// ---- FNV-1a snapshot checksum: bytes.hpp:14-22, tensor_bytes.hpp:26-29 ----
uint64_t fnv1a64(const void* data, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= static_cast<uint64_t>(p[i]);
        h *= 0x100000001b3ull;
    }
    return h;
}
uint64_t matrix_checksum(const Matd& m) { return fnv1a64(m.d.data(), m.d.size() * sizeof(double)); }

// ---- precond.cpp ------------------------------------------------------------
void validate(const asg_optimizer_config& c) {  // precond.cpp:34-42
    if (c.precondition_frequency < 1) throw Error(ASG_ERR_CONFIG_INVALID, "precondition_frequency must be >= 1");
    if (c.beta1 < 0.0 || c.beta1 >= 1.0 || c.beta2 < 0.0 || c.beta2 >= 1.0)
        throw Error(ASG_ERR_CONFIG_INVALID, "betas must lie in [0, 1)");
    if (c.lr < 0.0 || c.eps <= 0.0 || c.damping < 0.0 || c.weight_decay < 0.0)
        throw Error(ASG_ERR_CONFIG_INVALID, "lr/eps/damping/weight_decay out of range");
    if (c.block_dim_limit < 1) throw Error(ASG_ERR_CONFIG_INVALID, "block_dim_limit must be >= 1");
}

asg_optimizer_config defaults_for(int method) {  // precond.cpp:44-62 (+ KL-Shampoo)
    asg_optimizer_config c{};
    c.method = method;
    c.lr = 1e-3;
    c.beta1 = 0.9;
    c.beta2 = 0.95;
    c.eps = 1e-8;
    c.weight_decay = 0.0;
    c.precondition_frequency = 10;
    c.accumulation = ASG_ACCUM_SUM;
    c.damping = 1e-8;
    c.block_dim_limit = 2048;
    switch (method) {
        case ASG_METHOD_ADAMW: c.beta2 = 0.999; c.accumulation = ASG_ACCUM_SUM; break;
        case ASG_METHOD_SHAMPOO: c.beta2 = 0.95; c.accumulation = ASG_ACCUM_SUM; break;
        case ASG_METHOD_SOAP: c.beta2 = 0.95; c.accumulation = ASG_ACCUM_EMA; break;
        case ASG_METHOD_KL_SHAMPOO: c.beta2 = 0.95; c.accumulation = ASG_ACCUM_EMA; break;
        default: throw Error(ASG_ERR_CONFIG_INVALID, "unknown optimizer method");
    }
    return c;
}

struct Block {  // PrecondBlock precond.hpp:63-75, create precond.cpp:84-110
    int64_t rows = 0, cols = 0;
    int method = ASG_METHOD_SHAMPOO;
    Matd factor_l, factor_r, inv_l, inv_r, kl_inv_l, kl_inv_r;
    EigenPair<double> basis_l, basis_r;
    Matd rotated_m, rotated_v;
    uint64_t version = 0;
    int64_t last_refresh_step = -1;
    int64_t moment_steps = 0;
    static Block create(int64_t nr, int64_t nc, int method) {
        Block b;
        b.rows = nr;
        b.cols = nc;
        b.method = method;
        // KL-Shampoo starts from identity statistics (its inverses feed the
        // next statistics, so a zero start with the reference's 1e-8 relative
        // damping amplifies rank-deficient directions by ~1e8); Shampoo/SOAP
        // start from zero as PrecondBlock::create does (precond.cpp:89-90).
        b.factor_l = method == ASG_METHOD_KL_SHAMPOO ? Matd::identity(nr) : Matd(nr, nr);
        b.factor_r = method == ASG_METHOD_KL_SHAMPOO ? Matd::identity(nc) : Matd(nc, nc);
        b.inv_l = Matd::identity(nr);
        b.inv_r = Matd::identity(nc);
        b.kl_inv_l = Matd::identity(nr);
        b.kl_inv_r = Matd::identity(nc);
        b.basis_l = EigenPair<double>::identity(nr);
        b.basis_r = EigenPair<double>::identity(nc);
        b.rotated_m = Matd(nr, nc);
        b.rotated_v = Matd(nr, nc);
        return b;
    }
};

struct Snapshot {  // FactorSnapshot precond.hpp:77-81
    Matd factor_l, factor_r;
    uint64_t checksum = 0;
};

struct Refresh {  // RefreshResult precond.hpp:83-87 (+ KL inverses)
    Matd inv_l, inv_r, kl_inv_l, kl_inv_r;
    EigenPair<double> basis_l, basis_r;
    bool soap = false;
    bool kl = false;
};

uint64_t snapshot_checksum(const Matd& l, const Matd& r) {  // precond.cpp:114-115
    const uint64_t hl = matrix_checksum(l);
    return matrix_checksum(r) ^ (hl * 0x9e3779b97f4a7c15ull);
}

Snapshot snapshot_factors(const Block& b) {  // precond.cpp:112-117
    Snapshot s{b.factor_l, b.factor_r, 0};
    s.checksum = snapshot_checksum(s.factor_l, s.factor_r);
    return s;
}

double relative_damping(const Matd& m, double damping) {  // precond.cpp:121-125
    const int64_t n = m.r;
    if (n == 0) return 0.0;
    double tr = 0.0;
    for (int64_t i = 0; i < n; ++i) tr += m(i, i);
    return damping * tr / static_cast<double>(n);
}

Refresh compute_refresh(const Snapshot& snap, const asg_optimizer_config& cfg) {  // precond.cpp:129-142
    Refresh out;
    if (cfg.method == ASG_METHOD_SOAP) {
        out.soap = true;
        out.basis_l = sym_eig(snap.factor_l);
        out.basis_r = sym_eig(snap.factor_r);
        out.inv_l = Matd::identity(snap.factor_l.r);
        out.inv_r = Matd::identity(snap.factor_r.r);
    } else if (cfg.method == ASG_METHOD_KL_SHAMPOO) {
        // KL-Shampoo: one eigh per side gives both L^-1/2 (update) and L^-1
        // (next statistics), with the reference's relative damping.
        out.kl = true;
        const Matd* f[2] = {&snap.factor_l, &snap.factor_r};
        Matd* root[2] = {&out.inv_l, &out.inv_r};
        Matd* inv[2] = {&out.kl_inv_l, &out.kl_inv_r};
        for (int side = 0; side < 2; ++side) {
            EigenPair<double> e = sym_eig(*f[side]);
            const double eps = relative_damping(*f[side], cfg.damping);
            const int64_t n = f[side]->r;
            std::vector<double> wr(static_cast<size_t>(n)), wi(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) {
                const double damped = e.values[static_cast<size_t>(i)] + eps;
                if (damped <= 0.0)
                    throw Error(ASG_ERR_NOT_PSD, "kl refresh: damped eigenvalue <= 0 at index " +
                                                     std::to_string(i));
                wr[static_cast<size_t>(i)] = std::pow(damped, -0.5);
                wi[static_cast<size_t>(i)] = 1.0 / damped;
            }
            *root[side] = reconstruct(e, wr);
            *inv[side] = reconstruct(e, wi);
        }
    } else {
        out.inv_l = inv_root(snap.factor_l, 4, relative_damping(snap.factor_l, cfg.damping));
        out.inv_r = inv_root(snap.factor_r, 4, relative_damping(snap.factor_r, cfg.damping));
    }
    return out;
}

void install_refresh(Block& b, Refresh&& r, int64_t step) {  // precond.cpp:144-164
    if (r.soap) {
        const Matd rot_l = matmul(r.basis_l.vectors.transpose(), b.basis_l.vectors);
        const Matd rot_r = matmul(r.basis_r.vectors.transpose(), b.basis_r.vectors);
        b.rotated_m = matmul(matmul(rot_l, b.rotated_m), rot_r.transpose());
        Matd rot_l2 = rot_l, rot_r2 = rot_r;
        for (double& x : rot_l2.d) x *= x;
        for (double& x : rot_r2.d) x *= x;
        b.rotated_v = matmul(matmul(rot_l2, b.rotated_v), rot_r2.transpose());
        b.basis_l = std::move(r.basis_l);
        b.basis_r = std::move(r.basis_r);
    } else {
        b.inv_l = std::move(r.inv_l);
        b.inv_r = std::move(r.inv_r);
        if (r.kl) {
            b.kl_inv_l = std::move(r.kl_inv_l);
            b.kl_inv_r = std::move(r.kl_inv_r);
        }
    }
    b.version += 1;
    b.last_refresh_step = step;
}

void check_shape(const Block& b, const Matd& g, const char* what) {
    if (g.r != b.rows || g.c != b.cols)
        throw Error(ASG_ERR_SHAPE_MISMATCH, std::string(what) + ": gradient shape mismatch");
}

void accumulate_factors(Block& b, const Matd& g, const asg_optimizer_config& cfg) {  // precond.cpp:173-189
    check_shape(b, g, "accumulate_factors");
    if (!g.all_finite()) throw Error(ASG_ERR_NON_FINITE, "accumulate_factors: non-finite gradient");
    Matd gl, gr;
    if (cfg.method == ASG_METHOD_KL_SHAMPOO) {
        // G R^-1 G^T / n and G^T L^-1 G / m with the installed inverses.
        gl = symmetrized(matmul(matmul(g, b.kl_inv_r), g.transpose()));
        gr = symmetrized(matmul(matmul(g.transpose(), b.kl_inv_l), g));
        for (double& x : gl.d) x /= static_cast<double>(b.cols);
        for (double& x : gr.d) x /= static_cast<double>(b.rows);
    } else {
        gl = gram_left(g);
        gr = gram_right(g);
    }
    if (cfg.accumulation == ASG_ACCUM_SUM) {
        for (size_t i = 0; i < gl.d.size(); ++i) b.factor_l.d[i] += gl.d[i];
        for (size_t i = 0; i < gr.d.size(); ++i) b.factor_r.d[i] += gr.d[i];
    } else {
        const double beta = cfg.beta2;
        for (size_t i = 0; i < gl.d.size(); ++i)
            b.factor_l.d[i] = beta * b.factor_l.d[i] + (1.0 - beta) * gl.d[i];
        for (size_t i = 0; i < gr.d.size(); ++i)
            b.factor_r.d[i] = beta * b.factor_r.d[i] + (1.0 - beta) * gr.d[i];
    }
}

Matd precondition_shampoo(const Block& b, const Matd& g) {  // precond.cpp:191-198
    if (b.version == 0)
        throw Error(ASG_ERR_STALE_UNINITIALIZED, "precondition_shampoo: no inverse installed");
    check_shape(b, g, "precondition_shampoo");
    return matmul(matmul(b.inv_l, g), b.inv_r);
}

Matd soap_scaled_step(Block& b, const Matd& g, const asg_optimizer_config& cfg) {  // precond.cpp:208-223
    check_shape(b, g, "precondition_soap");
    const Matd rotated = matmul(matmul(b.basis_l.vectors.transpose(), g), b.basis_r.vectors);
    b.moment_steps += 1;
    const double t = static_cast<double>(b.moment_steps);
    for (size_t i = 0; i < rotated.d.size(); ++i) {
        b.rotated_m.d[i] = cfg.beta1 * b.rotated_m.d[i] + (1.0 - cfg.beta1) * rotated.d[i];
        b.rotated_v.d[i] =
            cfg.beta2 * b.rotated_v.d[i] + (1.0 - cfg.beta2) * (rotated.d[i] * rotated.d[i]);
    }
    const double bc1 = 1.0 - std::pow(cfg.beta1, t);
    const double bc2 = 1.0 - std::pow(cfg.beta2, t);
    Matd scaled(b.rows, b.cols);
    for (size_t i = 0; i < scaled.d.size(); ++i) {
        const double m_hat = b.rotated_m.d[i] / bc1;
        const double v_hat = b.rotated_v.d[i] / bc2;
        scaled.d[i] = m_hat / (std::sqrt(v_hat) + cfg.eps);
    }
    return matmul(matmul(b.basis_l.vectors, scaled), b.basis_r.vectors.transpose());
}

Matd precondition_soap(Block& b, const Matd& g, const asg_optimizer_config& cfg) {  // precond.cpp:200-206
    if (b.version == 0)
        throw Error(ASG_ERR_STALE_UNINITIALIZED, "precondition_soap: no basis installed");
    return soap_scaled_step(b, g, cfg);
}

struct Adam {  // AdamState precond.hpp:122-126
    Matd m, v;
    int64_t t = 0;
};

Matd adamw_step(Adam& st, const Matd& g, const asg_optimizer_config& cfg) {  // precond.cpp:229-242
    if (!g.all_finite()) throw Error(ASG_ERR_NON_FINITE, "adamw_step: non-finite gradient");
    if (g.r != st.m.r || g.c != st.m.c) throw Error(ASG_ERR_SHAPE_MISMATCH, "adamw_step: gradient shape mismatch");
    st.t += 1;
    const double t = static_cast<double>(st.t);
    const double bc1 = 1.0 - std::pow(cfg.beta1, t);
    const double bc2 = 1.0 - std::pow(cfg.beta2, t);
    Matd out(g.r, g.c);
    for (size_t i = 0; i < g.d.size(); ++i) {
        st.m.d[i] = cfg.beta1 * st.m.d[i] + (1.0 - cfg.beta1) * g.d[i];
        st.v.d[i] = cfg.beta2 * st.v.d[i] + (1.0 - cfg.beta2) * (g.d[i] * g.d[i]);
        out.d[i] = (st.m.d[i] / bc1) / (std::sqrt(st.v.d[i] / bc2) + cfg.eps);
    }
    return out;
}

void apply_update(Matd& theta, const Matd& update, const asg_optimizer_config& cfg,
                  double lr_scale) {  // precond.cpp:244-251
    if (theta.r != update.r || theta.c != update.c) throw Error(ASG_ERR_SHAPE_MISMATCH, "apply_update: shape mismatch");
    if (!update.all_finite()) throw Error(ASG_ERR_NON_FINITE, "apply_update: non-finite update");
    const double lr = cfg.lr * lr_scale;
    for (size_t i = 0; i < theta.d.size(); ++i)
        theta.d[i] -= lr * (update.d[i] + cfg.weight_decay * theta.d[i]);
}

// Cold-start rule + precondition (harness.cpp:455-466).
Matd step_update(Block& b, const Matd& g, const asg_optimizer_config& cfg) {
    if (b.version == 0) {
        if (cfg.method == ASG_METHOD_SOAP) return soap_scaled_step(b, g, cfg);
        return g;
    }
    if (cfg.method == ASG_METHOD_SOAP) return precondition_soap(b, g, cfg);
    return precondition_shampoo(b, g);
}

// ---- ShadowScheduler rules (asyncsched.cpp:108-221, 268-286) ---------------
struct Pending {
    int64_t dispatch_step = 0;
    double dispatch_sim_us = 0, completion_sim_us = 0;
    uint64_t snapshot_checksum = 0;
    Refresh result;  // computed at dispatch: the job is pure over its snapshot
};

struct Freshness {
    uint64_t installed_version = 0;
    int64_t dispatch_step_of_pending = -1;
    int64_t last_install_step = -1;
    int64_t installed_snapshot_step = -1;
};

struct Sched {
    asg_optimizer_config opt{};
    asg_scheduler_config cfg{};
    double now_us = 0.0;
    std::mt19937_64 jitter_rng;
    std::map<int64_t, Pending> pending;  // keyed by block id (index)
    std::map<int64_t, Freshness> fresh;
    asg_pool_stats stats{};
    std::vector<asg_event> events;
    bool pool_down = false;

    Sched(const asg_optimizer_config& o, const asg_scheduler_config& c, uint64_t seed)
        : opt(o), cfg(c), jitter_rng(seed * 0x9e3779b97f4a7c15ull + 0x2545f4914f6cdd1dull) {
        if (cfg.staleness_S < 0) throw Error(ASG_ERR_CONFIG_INVALID, "staleness_S must be >= 0");
        if (cfg.pf < 1) throw Error(ASG_ERR_CONFIG_INVALID, "pf must be >= 1");
    }
    void emit(int64_t step, int kind, int64_t block, uint64_t version, double t) {
        asg_event e{};
        e.step = step;
        e.kind = kind;
        e.block = block;
        e.version = version;
        e.t_us = t;
        events.push_back(e);
    }
    bool maybe_dispatch(Block& b, int64_t id, int64_t step) {  // asyncsched.cpp:108-142
        if (step % cfg.pf != 0) return false;
        if (pending.count(id)) {
            stats.coalesced += 1;
            return false;
        }
        if (pool_down) throw Error(ASG_ERR_WORKER_POOL_DOWN, "asyncsched: dispatch after pool stop");
        Snapshot snap = snapshot_factors(b);
        double cost_steps = cfg.inject_job_delay_steps;
        if (cfg.inject_job_delay_jitter_steps > 0.0) {
            std::uniform_real_distribution<double> dist(0.0, cfg.inject_job_delay_jitter_steps);
            cost_steps += dist(jitter_rng);
        }
        Pending p;
        p.dispatch_step = step;
        p.dispatch_sim_us = now_us;
        p.completion_sim_us = now_us + cost_steps * cfg.step_compute_us;
        p.snapshot_checksum = snap.checksum;
        if (snapshot_checksum(snap.factor_l, snap.factor_r) != p.snapshot_checksum)
            throw Error(ASG_ERR_AUDIT, "asyncsched: snapshot mutated");
        p.result = compute_refresh(snap, opt);
        emit(step, ASG_EV_DISPATCH, id, b.version, now_us);
        fresh[id].dispatch_step_of_pending = step;
        pending.emplace(id, std::move(p));
        stats.dispatched += 1;
        return true;
    }
    void install(Block& b, int64_t id, Pending p, int64_t step) {  // asyncsched.cpp:144-189
        stats.completed += 1;
        emit(p.dispatch_step, ASG_EV_JOB_START, id, b.version, p.dispatch_sim_us);
        emit(step, ASG_EV_JOB_DONE, id, b.version, p.completion_sim_us);
        install_refresh(b, std::move(p.result), step);
        now_us += cfg.install_cost_us;
        Freshness& rec = fresh[id];
        rec.installed_version = b.version;
        rec.last_install_step = step;
        rec.installed_snapshot_step = p.dispatch_step;
        rec.dispatch_step_of_pending = -1;
        emit(step, ASG_EV_INSTALL, id, b.version, now_us);
        stats.installed += 1;
    }
    double barrier(Block& b, int64_t id, int64_t step) {  // asyncsched.cpp:191-221
        auto it = pending.find(id);
        if (it == pending.end()) return 0.0;
        const int64_t age = step - it->second.dispatch_step;
        const bool stale_consumer =
            b.version > 0 &&
            step - fresh[id].installed_snapshot_step > (cfg.staleness_S + 1) * cfg.pf;
        const bool wait = cfg.staleness_S == 0 || age > cfg.staleness_S || stale_consumer;
        if (!wait) return 0.0;
        if (pool_down) throw Error(ASG_ERR_WORKER_POOL_DOWN, "asyncsched: barrier with pool down");
        const double waited = std::max(0.0, it->second.completion_sim_us - now_us);
        emit(step, ASG_EV_BARRIER_WAIT_BEGIN, id, b.version, now_us);
        now_us += waited;
        Pending taken = std::move(it->second);
        pending.erase(it);
        install(b, id, std::move(taken), step);
        emit(step, ASG_EV_BARRIER_WAIT_END, id, b.version, now_us);
        stats.barrier_waits += 1;
        stats.wait_total_us += waited;
        return waited;
    }
    void step_end(Block** blocks, const int64_t* ids, int64_t n, int64_t step) {  // asyncsched.cpp:268-286
        // Ids are installed in ascending order (std::sort of block id strings
        // at asyncsched.cpp:276; callers that need the same order pass ids
        // whose numeric order matches).
        std::vector<int64_t> ready;
        for (auto& kv : pending)
            if (kv.second.completion_sim_us <= now_us) ready.push_back(kv.first);
        for (int64_t id : ready) {
            Block* b = nullptr;
            for (int64_t k = 0; k < n; ++k)
                if (ids[k] == id) b = blocks[k];
            if (!b) continue;
            Pending p = std::move(pending[id]);
            pending.erase(id);
            install(*b, id, std::move(p), step);
        }
    }
};

}  // namespace orc

// ============================================================================
// extern "C" API (ctypes). Matrices are row-major double arrays.
// ============================================================================
using namespace orc;

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return ASG_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return ASG_ERR_INVALID_ARGUMENT;
    }
}

Matd from_ptr(const double* p, int64_t r, int64_t c) {
    Matd m(r, c);
    if (r * c > 0) std::memcpy(m.d.data(), p, sizeof(double) * static_cast<size_t>(r * c));
    return m;
}
void to_ptr(const Matd& m, double* p) {
    if (!m.d.empty()) std::memcpy(p, m.d.data(), sizeof(double) * m.d.size());
}

struct OrcBlock {
    Block b;
};
struct OrcAdam {
    Adam a;
};
struct OrcSched {
    std::unique_ptr<Sched> s;
};

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_last_error.c_str(); }

int orc_random_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    return guard([&] { to_ptr(random_matrix(rows, cols, seed), out); });
}
int orc_random_spd(int64_t dim, uint64_t seed, double ridge, double* out) {
    return guard([&] { to_ptr(random_spd(dim, seed, ridge), out); });
}
int orc_matmul(const double* a, const double* b, int64_t m, int64_t k, int64_t n, double* out) {
    return guard([&] { to_ptr(matmul(from_ptr(a, m, k), from_ptr(b, k, n)), out); });
}
int orc_gram_left(const double* g, int64_t r, int64_t c, double* out) {
    return guard([&] { to_ptr(gram_left(from_ptr(g, r, c)), out); });
}
int orc_gram_right(const double* g, int64_t r, int64_t c, double* out) {
    return guard([&] { to_ptr(gram_right(from_ptr(g, r, c)), out); });
}
int orc_sym_eig(const double* a, int64_t n, double* values, double* vectors) {
    return guard([&] {
        EigenPair<double> e = sym_eig(from_ptr(a, n, n));
        std::copy(e.values.begin(), e.values.end(), values);
        to_ptr(e.vectors, vectors);
    });
}
int orc_inv_root(const double* a, int64_t n, int root_order, double damping, double* out) {
    return guard([&] { to_ptr(inv_root(from_ptr(a, n, n), root_order, damping), out); });
}
// Extended-precision oracle (test_util.hpp:32-37): same algorithm in long double.
int orc_inv_root_xp(const double* a, int64_t n, int root_order, double damping, double* out) {
    return guard([&] {
        Mat<long double> m(n, n);
        for (int64_t i = 0; i < n * n; ++i) m.d[static_cast<size_t>(i)] = a[i];
        Mat<long double> r = inv_root<long double>(m, root_order, (long double)damping);
        for (int64_t i = 0; i < n * n; ++i) out[i] = static_cast<double>(r.d[static_cast<size_t>(i)]);
    });
}
int orc_pack_spd(const double* a, int64_t n, double* packed) {  // densela.hpp:124-135
    return guard([&] {
        int64_t k = 0;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j <= i; ++j) packed[k++] = a[i * n + j];
    });
}
int orc_unpack_spd(const double* packed, int64_t n, double* a) {  // densela.hpp:86-98,137-142
    return guard([&] {
        int64_t k = 0;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j <= i; ++j) {
                a[i * n + j] = packed[k];
                a[j * n + i] = packed[k];
                ++k;
            }
    });
}
int orc_checksum(const double* a, int64_t count, uint64_t* out) {
    return guard([&] { *out = fnv1a64(a, sizeof(double) * static_cast<size_t>(count)); });
}

int orc_defaults_for(int method, asg_optimizer_config* out) {
    return guard([&] { *out = defaults_for(method); });
}
int orc_validate(const asg_optimizer_config* c) { return guard([&] { validate(*c); }); }

void* orc_block_create(int64_t rows, int64_t cols, int method) {
    auto* b = new OrcBlock;
    b->b = Block::create(rows, cols, method);
    return b;
}
void orc_block_free(void* h) { delete static_cast<OrcBlock*>(h); }
void* orc_block_clone(void* h) { return new OrcBlock(*static_cast<OrcBlock*>(h)); }

int orc_block_get(void* h, int role, double* out) {
    return guard([&] {
        Block& b = static_cast<OrcBlock*>(h)->b;
        switch (role) {
            case ASG_ROLE_FACTOR_L: to_ptr(b.factor_l, out); break;
            case ASG_ROLE_FACTOR_R: to_ptr(b.factor_r, out); break;
            case ASG_ROLE_INV_L: to_ptr(b.inv_l, out); break;
            case ASG_ROLE_INV_R: to_ptr(b.inv_r, out); break;
            case ASG_ROLE_BASIS_L: to_ptr(b.basis_l.vectors, out); break;
            case ASG_ROLE_BASIS_R: to_ptr(b.basis_r.vectors, out); break;
            case ASG_ROLE_ROTATED_M: to_ptr(b.rotated_m, out); break;
            case ASG_ROLE_ROTATED_V: to_ptr(b.rotated_v, out); break;
            case ASG_ROLE_KL_INV_L: to_ptr(b.kl_inv_l, out); break;
            case ASG_ROLE_KL_INV_R: to_ptr(b.kl_inv_r, out); break;
            case ASG_ROLE_EIGVALS_L: std::copy(b.basis_l.values.begin(), b.basis_l.values.end(), out); break;
            case ASG_ROLE_EIGVALS_R: std::copy(b.basis_r.values.begin(), b.basis_r.values.end(), out); break;
            default: throw Error(ASG_ERR_INVALID_ARGUMENT, "unknown role");
        }
    });
}
int orc_block_set(void* h, int role, const double* in) {
    return guard([&] {
        Block& b = static_cast<OrcBlock*>(h)->b;
        const int64_t m = b.rows, n = b.cols;
        switch (role) {
            case ASG_ROLE_FACTOR_L: b.factor_l = from_ptr(in, m, m); break;
            case ASG_ROLE_FACTOR_R: b.factor_r = from_ptr(in, n, n); break;
            case ASG_ROLE_INV_L: b.inv_l = from_ptr(in, m, m); break;
            case ASG_ROLE_INV_R: b.inv_r = from_ptr(in, n, n); break;
            case ASG_ROLE_BASIS_L: b.basis_l.vectors = from_ptr(in, m, m); break;
            case ASG_ROLE_BASIS_R: b.basis_r.vectors = from_ptr(in, n, n); break;
            case ASG_ROLE_ROTATED_M: b.rotated_m = from_ptr(in, m, n); break;
            case ASG_ROLE_ROTATED_V: b.rotated_v = from_ptr(in, m, n); break;
            case ASG_ROLE_KL_INV_L: b.kl_inv_l = from_ptr(in, m, m); break;
            case ASG_ROLE_KL_INV_R: b.kl_inv_r = from_ptr(in, n, n); break;
            case ASG_ROLE_EIGVALS_L: b.basis_l.values.assign(in, in + m); break;
            case ASG_ROLE_EIGVALS_R: b.basis_r.values.assign(in, in + n); break;
            default: throw Error(ASG_ERR_INVALID_ARGUMENT, "unknown role");
        }
    });
}
int orc_block_counters(void* h, uint64_t* version, int64_t* last_refresh_step, int64_t* moment_steps) {
    Block& b = static_cast<OrcBlock*>(h)->b;
    *version = b.version;
    *last_refresh_step = b.last_refresh_step;
    *moment_steps = b.moment_steps;
    return ASG_OK;
}
int orc_block_set_counters(void* h, uint64_t version, int64_t last_refresh_step, int64_t moment_steps) {
    Block& b = static_cast<OrcBlock*>(h)->b;
    b.version = version;
    b.last_refresh_step = last_refresh_step;
    b.moment_steps = moment_steps;
    return ASG_OK;
}
int orc_accumulate(void* h, const double* g, const asg_optimizer_config* cfg) {
    return guard([&] {
        Block& b = static_cast<OrcBlock*>(h)->b;
        accumulate_factors(b, from_ptr(g, b.rows, b.cols), *cfg);
    });
}
int orc_snapshot_checksum(void* h, uint64_t* out) {
    return guard([&] { *out = snapshot_factors(static_cast<OrcBlock*>(h)->b).checksum; });
}
int orc_refresh_inverse(void* h, const asg_optimizer_config* cfg, int64_t step) {  // precond.cpp:166-171
    return guard([&] {
        Block& b = static_cast<OrcBlock*>(h)->b;
        install_refresh(b, compute_refresh(snapshot_factors(b), *cfg), step);
    });
}
// compute_refresh over a snapshot of `src`, installed into `dst`
// (models a refresh dispatched earlier and installed now).
int orc_refresh_from(void* dst, void* src, const asg_optimizer_config* cfg, int64_t step) {
    return guard([&] {
        Block& d = static_cast<OrcBlock*>(dst)->b;
        Block& s = static_cast<OrcBlock*>(src)->b;
        install_refresh(d, compute_refresh(snapshot_factors(s), *cfg), step);
    });
}
int orc_precondition_shampoo(void* h, const double* g, double* out) {
    return guard([&] {
        Block& b = static_cast<OrcBlock*>(h)->b;
        to_ptr(precondition_shampoo(b, from_ptr(g, b.rows, b.cols)), out);
    });
}
int orc_precondition_soap(void* h, const double* g, const asg_optimizer_config* cfg, double* out) {
    return guard([&] {
        Block& b = static_cast<OrcBlock*>(h)->b;
        to_ptr(precondition_soap(b, from_ptr(g, b.rows, b.cols), *cfg), out);
    });
}
int orc_soap_scaled_step(void* h, const double* g, const asg_optimizer_config* cfg, double* out) {
    return guard([&] {
        Block& b = static_cast<OrcBlock*>(h)->b;
        to_ptr(soap_scaled_step(b, from_ptr(g, b.rows, b.cols), *cfg), out);
    });
}
int orc_step_update(void* h, const double* g, const asg_optimizer_config* cfg, double* out) {
    return guard([&] {
        Block& b = static_cast<OrcBlock*>(h)->b;
        to_ptr(step_update(b, from_ptr(g, b.rows, b.cols), *cfg), out);
    });
}
int orc_apply_update(double* theta, const double* update, int64_t r, int64_t c,
                     const asg_optimizer_config* cfg, double lr_scale) {
    return guard([&] {
        Matd t = from_ptr(theta, r, c);
        apply_update(t, from_ptr(update, r, c), *cfg, lr_scale);
        to_ptr(t, theta);
    });
}
int orc_replicated_state(void* h, double* flat) {  // precond.cpp:253-265
    return guard([&] {
        Block& b = static_cast<OrcBlock*>(h)->b;
        const bool soap = b.method == ASG_METHOD_SOAP;
        to_ptr(soap ? b.basis_l.vectors : b.inv_l, flat);
        to_ptr(soap ? b.basis_r.vectors : b.inv_r, flat + b.rows * b.rows);
    });
}

void* orc_adam_create(int64_t rows, int64_t cols) {
    auto* a = new OrcAdam;
    a->a.m = Matd(rows, cols);
    a->a.v = Matd(rows, cols);
    return a;
}
void orc_adam_free(void* h) { delete static_cast<OrcAdam*>(h); }
int orc_adamw_step(void* h, const double* g, const asg_optimizer_config* cfg, double* out) {
    return guard([&] {
        Adam& a = static_cast<OrcAdam*>(h)->a;
        to_ptr(adamw_step(a, from_ptr(g, a.m.r, a.m.c), *cfg), out);
    });
}

// --- harness helpers (harness.cpp:219-229) ---
double orc_clip_scale(const double* flat, int64_t n, double clip_norm) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += flat[i] * flat[i];
    const double norm = std::sqrt(acc);
    if (norm <= clip_norm || norm == 0.0) return 1.0;
    return clip_norm / norm;
}
double orc_warmup_scale(int64_t step, int64_t total_steps) {
    const int64_t warmup = std::max<int64_t>(1, total_steps / 20);
    if (step + 1 >= warmup) return 1.0;
    return static_cast<double>(step + 1) / static_cast<double>(warmup);
}

// --- scheduler ---
void* orc_sched_create(const asg_optimizer_config* opt, const asg_scheduler_config* cfg, uint64_t seed) {
    try {
        auto* s = new OrcSched;
        s->s = std::make_unique<Sched>(*opt, *cfg, seed);
        return s;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return nullptr;
    }
}
void orc_sched_free(void* h) { delete static_cast<OrcSched*>(h); }
int orc_sched_clock_advance(void* h, double us) {
    static_cast<OrcSched*>(h)->s->now_us += us;
    return ASG_OK;
}
int orc_sched_maybe_dispatch(void* h, void* blk, int64_t id, int64_t step, int* dispatched) {
    return guard([&] {
        *dispatched = static_cast<OrcSched*>(h)->s->maybe_dispatch(static_cast<OrcBlock*>(blk)->b, id, step);
    });
}
int orc_sched_barrier(void* h, void* blk, int64_t id, int64_t step, double* waited) {
    return guard([&] {
        *waited = static_cast<OrcSched*>(h)->s->barrier(static_cast<OrcBlock*>(blk)->b, id, step);
    });
}
int orc_sched_step_end(void* h, void** blks, const int64_t* ids, int64_t n, int64_t step) {
    return guard([&] {
        std::vector<Block*> bs(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) bs[static_cast<size_t>(i)] = &static_cast<OrcBlock*>(blks[i])->b;
        static_cast<OrcSched*>(h)->s->step_end(bs.data(), ids, n, step);
    });
}
int orc_sched_stats(void* h, asg_pool_stats* out) {
    Sched& s = *static_cast<OrcSched*>(h)->s;
    *out = s.stats;
    out->pending = static_cast<int32_t>(s.pending.size());
    out->queue_depth = 0;
    return ASG_OK;
}
int orc_sched_freshness(void* h, int64_t id, asg_freshness* out) {
    Sched& s = *static_cast<OrcSched*>(h)->s;
    auto it = s.fresh.find(id);
    if (it == s.fresh.end()) {
        g_last_error = "asyncsched: no freshness record";
        return ASG_ERR_MISSING_KEY;
    }
    out->installed_version = it->second.installed_version;
    out->dispatch_step_of_pending = it->second.dispatch_step_of_pending;
    out->last_install_step = it->second.last_install_step;
    out->installed_snapshot_step = it->second.installed_snapshot_step;
    return ASG_OK;
}
int64_t orc_sched_events(void* h, asg_event* out, int64_t cap) {
    Sched& s = *static_cast<OrcSched*>(h)->s;
    const int64_t n = static_cast<int64_t>(s.events.size());
    for (int64_t i = 0; i < std::min(n, cap); ++i) out[i] = s.events[static_cast<size_t>(i)];
    return n;
}
int orc_sched_stop_pool(void* h) {
    static_cast<OrcSched*>(h)->s->pool_down = true;
    return ASG_OK;
}

// Refresh of many blocks on a pool of `threads` host threads, as the reference
// runs compute_refresh on its WorkerPool (harness.cpp:312-316,
// asyncsched.cpp:129). Used only by the CPU-baseline timing.
int orc_refresh_many(void** blks, int64_t n, const asg_optimizer_config* cfg, int64_t step, int threads) {
    return guard([&] {
        std::vector<int> codes(static_cast<size_t>(n), ASG_OK);
        std::vector<std::thread> pool;
        const int t = std::max(1, threads);
        for (int w = 0; w < t; ++w)
            pool.emplace_back([&, w] {
                for (int64_t i = w; i < n; i += t) {
                    try {
                        Block& b = static_cast<OrcBlock*>(blks[i])->b;
                        install_refresh(b, compute_refresh(snapshot_factors(b), *cfg), step);
                    } catch (const Error& e) {
                        codes[static_cast<size_t>(i)] = e.code;
                    }
                }
            });
        for (auto& th : pool) th.join();
        for (int c : codes)
            if (c != ASG_OK) throw Error(c, "orc_refresh_many: a refresh failed");
    });
}

}  // extern "C"
