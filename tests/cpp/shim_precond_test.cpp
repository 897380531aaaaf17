// SPDX-License-Identifier: Apache-2.0
//
// Replays reference test bodies (proj/tests/precond_test.cpp) through the C++
// shim include/asopt_b200.hpp against the GPU library. Built by
// tests/test_cpp_shim.py (g++, links libasteria_b200.so); run on a B200.
//
// The reference checks fp64 results at 1e-10..1e-14; here the state is fp32
// (3xTF32 tensor-core products), so the stated tolerances of DESIGN.md §4 apply:
// exact where the reference is exact and the fp32 value is exact too (identity
// factors, powers of two), ~1e-6 relative otherwise.
#include <cmath>
#include <cstdio>
#include <random>

#include "asopt_b200.hpp"

using namespace asopt::b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_fail;                                                            \
            std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        bool ok_ = false;                                                        \
        try {                                                                    \
            (void)(expr);                                                        \
        } catch (const type&) {                                                  \
            ok_ = true;                                                          \
        } catch (...) {                                                          \
        }                                                                        \
        if (!ok_) {                                                              \
            ++g_fail;                                                            \
            std::fprintf(stderr, "%s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #type); \
        }                                                                        \
    } while (0)

// test_util.hpp:10-17 restated: mt19937_64 + std::normal_distribution.
static Matd random_matrix(int64_t r, int64_t c, uint64_t seed) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> d(0.0, 1.0);
    Matd m(r, c);
    for (double& x : m.data) x = d(gen);
    return m;
}

static double maxabs_diff(const Matd& a, const Matd& b) {
    double m = 0.0;
    for (size_t i = 0; i < a.data.size(); ++i) m = std::max(m, std::fabs(a.data[i] - b.data[i]));
    return m;
}

static Matd scaled_identity(int64_t n, double c) {
    Matd m = Matd::Identity(n, n);
    for (double& x : m.data) x *= c;
    return m;
}

static OptimizerConfig shampoo_cfg() {
    OptimizerConfig c = OptimizerConfig::defaults_for(Method::Shampoo);
    c.damping = 0.0;
    return c;
}

int main() {
    // precond_test.cpp:28-49 — partition tiling
    {
        auto v = partition_param("w", 3000, 500, 2048);
        CHECK(v.size() == 2);
        CHECK(v[0].rows() == 2048 && v[1].rows() == 952 && v[1].cols() == 500);
        CHECK(v[1].id() == "w[2048:3000,0:500]");
        auto sq = partition_param("w", 5000, 5000, 2048);
        CHECK(sq.size() == 9);
        CHECK(sq[8].rows() == 904 && sq[8].cols() == 904);
    }
    // precond_test.cpp:72-88 — accumulate Sum / EMA
    {
        auto cfg = shampoo_cfg();
        PrecondBlock b(2, 2, cfg);
        accumulate_factors(b, Matd::Identity(2, 2), cfg);
        CHECK(maxabs_diff(b.factor_l(), Matd::Identity(2, 2)) == 0.0);
        OptimizerConfig ema = cfg;
        ema.accumulation = Accumulation::Ema;
        ema.beta2 = 0.9;
        PrecondBlock be(2, 2, ema);
        Matd g = Matd::Zero(2, 2);
        g(0, 0) = g(1, 1) = std::sqrt(10.0);
        accumulate_factors(be, g, ema);
        CHECK(std::fabs(be.factor_l()(0, 0) - 1.0) < 1e-6);
        CHECK(std::fabs(be.factor_l()(1, 1) - 1.0) < 1e-6);
    }
    // precond_test.cpp:107-121 — refresh: identity and scalar root
    {
        auto cfg = shampoo_cfg();
        PrecondBlock b(2, 2, cfg);
        b.set(ASG_ROLE_FACTOR_L, Matd::Identity(2, 2));
        b.set(ASG_ROLE_FACTOR_R, Matd::Identity(2, 2));
        PrecondBlock r = refresh_inverse(b, cfg, 7);
        CHECK(r.version() == 1);
        CHECK(r.last_refresh_step() == 7);
        CHECK(b.version() == 0);  // pure over the input block
        CHECK(maxabs_diff(r.inv_l(), Matd::Identity(2, 2)) < 1e-7);
        b.set(ASG_ROLE_FACTOR_L, scaled_identity(2, 16.0));
        PrecondBlock r2 = refresh_inverse(b, cfg, 8);
        CHECK(maxabs_diff(r2.inv_l(), scaled_identity(2, 0.5)) < 1e-7);
        CHECK(maxabs_diff(r2.inv_r(), Matd::Identity(2, 2)) < 1e-7);
    }
    // precond_test.cpp:123-137 — versions monotonic
    {
        auto cfg = shampoo_cfg();
        cfg.damping = 1e-8;
        PrecondBlock b(4, 4, cfg);
        accumulate_factors(b, random_matrix(4, 4, 11), cfg);
        const Matd before = b.factor_l();
        refresh_inverse_inplace(b, cfg, 3);
        CHECK(maxabs_diff(b.factor_l(), before) == 0.0);
        CHECK(b.version() == 1);
        refresh_inverse_inplace(b, cfg, 13);
        CHECK(b.version() == 2 && b.last_refresh_step() == 13);
    }
    // precond_test.cpp:166-180 — Shampoo identity / diagonal
    {
        auto cfg = shampoo_cfg();
        PrecondBlock b(2, 2, cfg);
        Matd g = Matd::Zero(2, 2);
        g(0, 0) = 2.0;
        g(1, 1) = 4.0;
        b.set_counters(1, -1, 0);  // identity inverses from create()
        CHECK(maxabs_diff(precondition_shampoo(b, g), g) == 0.0);
        PrecondBlock b2(2, 2, cfg);
        accumulate_factors(b2, g, cfg);
        b2 = refresh_inverse(b2, cfg, 0);
        Matd t = precondition_shampoo(b2, g);
        CHECK(std::fabs(t(0, 0) - 1.0) < 1e-6 && std::fabs(t(1, 1) - 1.0) < 1e-6);
    }
    // precond_test.cpp:193-199 — StaleUninitialized
    {
        PrecondBlock b(2, 2, shampoo_cfg());
        CHECK_THROWS_AS(precondition_shampoo(b, Matd::Zero(2, 2)), StaleUninitializedError);
        auto scfg = OptimizerConfig::defaults_for(Method::Soap);
        PrecondBlock bs(2, 2, scfg);
        CHECK_THROWS_AS(precondition_soap(bs, Matd::Zero(2, 2), scfg), StaleUninitializedError);
    }
    // precond_test.cpp:201-212 — scalar factors: c^-1/2 G
    {
        auto cfg = shampoo_cfg();
        for (double c : {0.25, 1.0, 9.0}) {
            PrecondBlock b(5, 3, cfg);
            b.set(ASG_ROLE_FACTOR_L, scaled_identity(5, c));
            b.set(ASG_ROLE_FACTOR_R, scaled_identity(3, c));
            refresh_inverse_inplace(b, cfg, 0);
            Matd g = random_matrix(5, 3, 31);
            Matd t = precondition_shampoo(b, g);
            Matd e = g;
            for (double& x : e.data) x *= std::pow(c, -0.5);
            CHECK(maxabs_diff(t, e) < 1e-6 * 3.0);
        }
    }
    // precond_test.cpp:214-224 — SOAP first step with identity bases is sign-like
    {
        auto cfg = OptimizerConfig::defaults_for(Method::Soap);
        cfg.beta1 = 0.0;
        PrecondBlock b(2, 3, cfg);
        b.set_counters(1, -1, 0);
        Matd g = random_matrix(2, 3, 13);
        for (double& x : g.data) x *= 10.0;
        Matd t = precondition_soap(b, g, cfg);
        for (int64_t i = 0; i < 2; ++i)
            for (int64_t j = 0; j < 3; ++j) CHECK(std::fabs(t(i, j) - (g(i, j) > 0 ? 1.0 : -1.0)) < 1e-5);
    }
    // precond_test.cpp:226-234 — zero gradient decays v by beta2
    {
        auto cfg = OptimizerConfig::defaults_for(Method::Soap);
        PrecondBlock b(2, 2, cfg);
        b.set_counters(1, -1, 0);
        b.set(ASG_ROLE_ROTATED_V, Matd(2, 2, 1.0));
        Matd t = precondition_soap(b, Matd::Zero(2, 2), cfg);
        double mx = 0.0;
        for (double x : t.data) mx = std::max(mx, std::fabs(x));
        CHECK(mx == 0.0);
        CHECK(maxabs_diff(b.rotated_v(), Matd(2, 2, cfg.beta2)) < 1e-7);
    }
    // config validation (precond.cpp:34-42)
    {
        auto cfg = shampoo_cfg();
        cfg.precondition_frequency = 0;
        CHECK_THROWS_AS(cfg.validate(), ConfigInvalidError);
    }
    // precond.hpp:90-98 split refresh: install(compute(snapshot)) == refresh_inverse,
    // compute is pure, the snapshot is isolated from later accumulation
    {
        auto cfg = OptimizerConfig::defaults_for(Method::Shampoo);
        PrecondBlock a(24, 16, cfg), b(24, 16, cfg);
        for (uint64_t s = 0; s < 3; ++s) {
            const Matd g = random_matrix(24, 16, 40 + s);
            accumulate_factors(a, g, cfg);
            accumulate_factors(b, g, cfg);
        }
        refresh_inverse_inplace(a, cfg, 3);
        FactorSnapshot snap = snapshot_factors(b);
        const uint64_t c0 = snap.checksum();
        accumulate_factors(b, random_matrix(24, 16, 50), cfg);  // after the snapshot
        CHECK(snap.checksum() == c0);
        RefreshResult r = compute_refresh(snap, cfg);
        CHECK(b.version() == 0);
        install_refresh(b, std::move(r), 3);
        CHECK(b.version() == 1 && b.last_refresh_step() == 3);
        CHECK(maxabs_diff(a.inv_l(), b.inv_l()) < 1e-6);
        CHECK(maxabs_diff(a.inv_r(), b.inv_r()) < 1e-6);
        // replicated_state round trip (precond.cpp:253-279)
        std::vector<double> flat = replicated_state(b, Method::Shampoo);
        CHECK(flat.size() == size_t(24 * 24 + 16 * 16));
        PrecondBlock c(24, 16, cfg);
        load_replicated_state(c, Method::Shampoo, flat);
        CHECK(maxabs_diff(c.inv_l(), b.inv_l()) == 0.0);
        flat.pop_back();
        CHECK_THROWS_AS(load_replicated_state(c, Method::Shampoo, flat), ShapeMismatchError);
    }
    // precond_test.cpp:283-342: AdamW direction and apply_update KATs
    {
        auto cfg = OptimizerConfig::defaults_for(Method::AdamW);
        AdamState st = AdamState::zeros(2, 2);
        Matd g(2, 2, 0.5);
        Matd d = adamw_step(st, g, cfg);  // first step: m^/sqrt(v^) = sign(g)
        for (double x : d.data) CHECK(std::fabs(x - 1.0) < 2e-5);  // fp32 moments; 1/(1-beta2) = 1000 scales their rounding
        Matd theta(2, 2, 1.0);
        cfg.weight_decay = 0.5;
        apply_update(theta, Matd(2, 2, 1.0), cfg, 2.0);  // 1 - lr*2*(1 + 0.5)
        for (double x : theta.data) CHECK(std::fabs(x - (1.0 - cfg.lr * 2.0 * 1.5)) < 1e-15);
        Matd bad(2, 2, 0.0);
        bad(1, 0) = std::nan("");
        CHECK_THROWS_AS(apply_update(theta, bad, cfg), NonFiniteError);
    }
    // densela_test.cpp:117-153: pack / unpack round trip
    {
        Matd m = random_matrix(5, 5, 60);
        for (int64_t i = 0; i < 5; ++i)
            for (int64_t j = 0; j < i; ++j) m(j, i) = m(i, j);
        std::vector<double> p = pack_spd(m);
        CHECK(p.size() == 15 && p[1] == m(1, 0) && p[2] == m(1, 1));
        CHECK(maxabs_diff(unpack_spd(p, 5), m) == 0.0);
        CHECK_THROWS_AS(unpack_spd(p, 4), LayoutMismatchError);
    }
    std::printf("shim_precond_test: %d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
