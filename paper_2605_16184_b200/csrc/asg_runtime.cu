// SPDX-License-Identifier: Apache-2.0
//
// Host runtime of the B200 Asteria optimizer step, behind the C-ABI of
// include/asteria_b200.h.
//
// A blockset holds the second-order state of every parameter block this rank
// owns, grouped by block shape into contiguous HBM slabs ([block][rows][cols])
// so that each GEMM of the step is ONE batched tcgen05 launch per shape group:
//
//   Shampoo     stats: L = b L + a G G^T, R = b R + a G^T G  (2 sym GEMMs)
//               update: Y = P_L G ; theta -= lr (Y P_R + wd theta)  (2 GEMMs)
//   SOAP        stats as Shampoo (EMA)
//               T = Q_L^T G ; Adam(T Q_R) -> S ; W^T = (S Q_R^T)^T ;
//               theta -= lr (Q_L W + wd theta)                     (4 GEMMs)
//   KL-Shampoo  X = G R^-1 ; L = b L + a/n X G^T ; Z^T = G^T L^-1 ;
//               R = b R + a/m G^T Z ; update as Shampoo with P = F^-1/2 (6 GEMMs)
//
// The refresh (snapshot -> fp64 eigh -> roots / bases) runs on a low-priority
// side stream under the reference's bounded-staleness rules
// (asyncsched.cpp:108-221,268-286), emulated exactly on a simulated clock
// (ASG_INSTALL_SIM_CLOCK) or driven by stream events (ASG_INSTALL_EVENT).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/asteria_b200.h"
#include "asg_eigh.cuh"
#include "asg_json.hpp"
#include "asg_kernels.cuh"

namespace asg {
namespace {

thread_local std::string g_err;

struct Fail {
    int code;
    std::string msg;
};

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess)                                                                \
            throw Fail{e_ == cudaErrorMemoryAllocation ? ASG_ERR_OUT_OF_MEMORY : ASG_ERR_CUDA, \
                       std::string(#x) + ": " + cudaGetErrorString(e_)};                      \
    } while (0)

template <class F>
int guard(F&& f) {
    try {
        f();
        return ASG_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return ASG_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ASG_ERR_INVALID_ARGUMENT;
    } catch (...) {  // nothing crosses the C-ABI
        g_err = "unknown exception";
        return ASG_ERR_INVALID_ARGUMENT;
    }
}

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// configuration (precond.cpp:34-62, config.cpp:121-149)
// ---------------------------------------------------------------------------
asg_optimizer_config defaults_for(int method) {
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
        case ASG_METHOD_ADAMW: c.beta2 = 0.999; break;
        case ASG_METHOD_SHAMPOO: break;
        case ASG_METHOD_SOAP:
        case ASG_METHOD_KL_SHAMPOO: c.accumulation = ASG_ACCUM_EMA; break;
        default: throw Fail{ASG_ERR_CONFIG_INVALID, "unknown optimizer method"};
    }
    return c;
}

void validate(const asg_optimizer_config& c) {
    if (c.method < ASG_METHOD_ADAMW || c.method > ASG_METHOD_KL_SHAMPOO)
        throw Fail{ASG_ERR_CONFIG_INVALID, "unknown optimizer method"};
    if (c.accumulation != ASG_ACCUM_SUM && c.accumulation != ASG_ACCUM_EMA)
        throw Fail{ASG_ERR_CONFIG_INVALID, "unknown accumulation mode"};
    if (c.precondition_frequency < 1) throw Fail{ASG_ERR_CONFIG_INVALID, "precondition_frequency must be >= 1"};
    if (c.beta1 < 0.0 || c.beta1 >= 1.0 || c.beta2 < 0.0 || c.beta2 >= 1.0)
        throw Fail{ASG_ERR_CONFIG_INVALID, "betas must lie in [0, 1)"};
    if (c.lr < 0.0 || c.eps <= 0.0 || c.damping < 0.0 || c.weight_decay < 0.0)
        throw Fail{ASG_ERR_CONFIG_INVALID, "lr/eps/damping/weight_decay out of range"};
    if (c.block_dim_limit < 1) throw Fail{ASG_ERR_CONFIG_INVALID, "block_dim_limit must be >= 1"};
}

asg_scheduler_config sched_defaults() {
    asg_scheduler_config s{};
    s.staleness_S = 5;
    s.pf = 10;
    s.pool_size = 0;
    s.drain_budget = 4;
    s.inject_job_delay_steps = 0.0;
    s.inject_job_delay_jitter_steps = 0.0;
    s.step_compute_us = 1000.0;
    s.install_cost_us = 0.0;
    s.install_mode = ASG_INSTALL_SIM_CLOCK;
    s.refresh_mode = ASG_REFRESH_F64;
    return s;
}

int method_from_string(const std::string& s) {
    if (s == "AdamW") return ASG_METHOD_ADAMW;
    if (s == "Shampoo") return ASG_METHOD_SHAMPOO;
    if (s == "SOAP") return ASG_METHOD_SOAP;
    if (s == "KL-Shampoo") return ASG_METHOD_KL_SHAMPOO;
    throw Fail{ASG_ERR_CONFIG_INVALID, "unknown optimizer method: " + s};
}

// ---------------------------------------------------------------------------
// blockset state
// ---------------------------------------------------------------------------
struct Unit {
    asg_block_spec spec{};
    bool adamw = false;
    int owner = 0;
    int group = -1, slot = -1;
    uint64_t version = 0;
    int64_t last_refresh_step = -1;
    int64_t moment_steps = 0;
    // shadow scheduler
    bool pending = false;
    int64_t dispatch_step = 0;
    double dispatch_sim = 0.0, completion_sim = 0.0;
    bool launched = false;  // refresh enqueued on the side stream
    bool needs_launch = false;  // dispatched, refresh not yet enqueued
    bool snap_preloaded = false;  // compute_refresh: the snapshot slot already holds the caller's snapshot
    bool warm_start = false;    // a previous eigenbasis exists (decided at dispatch)
    cudaEvent_t done = nullptr;
    bool has_fresh = false;
    asg_freshness fresh{0, -1, -1, -1};
    // AdamW state (1-D parameters)
    float *am = nullptr, *av = nullptr;
    int64_t adam_t = 0;
    double cost = 0.0;
};

struct Group {
    int m = 0, n = 0, M = 0, N = 0, nb = 0;
    std::vector<int> units;
    float *L = nullptr, *R = nullptr, *snapL = nullptr, *snapR = nullptr;
    float *Gh = nullptr, *Gl = nullptr, *GTh = nullptr, *GTl = nullptr;
    float *Th = nullptr, *Tl = nullptr, *Sh = nullptr, *Sl = nullptr;
    // Shampoo: P = F^-1/4 ; KL: P = F^-1/2 (active + shadow). KL-Shampoo's
    // F^-1 is never stored: it enters the statistics only as G F_R^-1 G^T =
    // (G P_R)(G P_R)^T and G^T F_L^-1 G = (P_L G)^T (P_L G) (group_stats)
    float *PLh = nullptr, *PLl = nullptr, *PRh = nullptr, *PRl = nullptr;
    float *sPLh = nullptr, *sPLl = nullptr, *sPRh = nullptr, *sPRl = nullptr;
    // KL-Shampoo: slot k of T holds V = P_L G for the block's current G and
    // roots (left there by group_stats); the update reuses it unless an
    // install or a new gradient intervened
    std::vector<uint8_t> v_ok;
    // 3XF16 (Shampoo / KL-Shampoo): the step's operands as fp16 (hi, lo) pairs
    // ([nb][rows][K] hi, then lo; 4 B per element) with per-block power-of-two
    // scales. G16 / GT16 reuse the G / G^T slabs; T16 (W or V), S16 (V^T), P16
    // (installed roots, converted at install; the fp32 roots stay for readers).
    uint16_t *G16 = nullptr, *GT16 = nullptr, *T16 = nullptr, *S16 = nullptr, *PL16 = nullptr, *PR16 = nullptr;
    float *gscale = nullptr, *tscale = nullptr, *sscale = nullptr, *plscale = nullptr, *prscale = nullptr;
    unsigned int *amax = nullptr, *amax2 = nullptr;  // per-block max |x| scratch
    unsigned int *pln1 = nullptr, *prn1 = nullptr;   // per-block 1-norm of the fp16 roots (float bits)
    unsigned int* amaxp = nullptr;  // previous step's max |G| per block (the predicted fp16 scale)
    int* gfix = nullptr;            // blocks whose predicted scale failed this step
    // SOAP
    float *QLh = nullptr, *QLl = nullptr, *QLTh = nullptr, *QLTl = nullptr;
    float *QRh = nullptr, *QRl = nullptr, *QRTh = nullptr, *QRTl = nullptr;
    float *mom_m = nullptr, *mom_v = nullptr;
    double *QL64 = nullptr, *QR64 = nullptr, *valsL = nullptr, *valsR = nullptr;
    double *sQL64 = nullptr, *sQR64 = nullptr, *svalsL = nullptr, *svalsR = nullptr;
    // Shampoo / KL-Shampoo: eigenvectors of the last refresh (warm start of the next)
    double *EL64 = nullptr, *ER64 = nullptr;
    // F32 refresh: Shampoo / KL basis as split tf32 pairs, row-major and transposed
    float *BLh = nullptr, *BLl = nullptr, *BLTh = nullptr, *BLTl = nullptr;
    float *BRh = nullptr, *BRl = nullptr, *BRTh = nullptr, *BRTl = nullptr;
    // F32 refresh, SOAP: shadow rotations J^T (new basis = Q_old J) per side
    float *sJLTh = nullptr, *sJLTl = nullptr, *sJRTh = nullptr, *sJRTl = nullptr;
    BlockRef* d_refs = nullptr;
    ApplyEntry* d_apply = nullptr;
    int2 *tilesM = nullptr, *tilesN = nullptr;
    int ntM = 0, ntN = 0;
    bool vec_grad = false;  // all gradient block rows 16-byte aligned (vectorised prep)
    int* d_status = nullptr;
    int* h_status = nullptr;  // pinned
    // F32 refresh: 1 where the eigensolve left the basis exactly unchanged (J = I);
    // such SOAP installs reduce to the eigenvalue copy
    int *d_identL = nullptr, *d_identR = nullptr, *h_identL = nullptr, *h_identR = nullptr;
};

}  // namespace
}  // namespace asg

struct asg_blockset {
    int device = 0;
    int num_sms = 148;
    asg_optimizer_config opt{};
    asg_scheduler_config sc{};
    int precision = ASG_PREC_3XTF32;
    int rank = 0, world = 1;
    std::vector<asg_param_desc> params;
    std::vector<asg::Unit> units;
    std::vector<asg::Group> groups;
    std::vector<void*> allocs;
    // F3: optional tiered store of the installed inverse state (asyncsched.cpp:164-184,223-267)
    asg_tierstore* store = nullptr;
    float* store_stage = nullptr;  // contiguous (hi | lo) staging of one installed root / basis
    size_t store_stage_floats = 0;
    struct QueuedPrefetch {
        std::string block_id;
        int32_t role;
        int unit;
        int64_t enqueue_step;
    };
    std::deque<QueuedPrefetch> queued_prefetches;
    // asg_synth_gradients: this rank's unit gradient views (bench input generation)
    asg::SynthBlock* d_synth = nullptr;
    int n_synth = 0;
    int synth_rows = 0, synth_cols = 0;
    size_t alloc_bytes = 0;      // every device allocation of the blockset
    size_t workspace_bytes = 0;  // of which: refresh / install workspace (alloc_workspace)
    std::vector<void*> host_allocs;
    cudaStream_t main = nullptr, side = nullptr;
    bool own_main = false;
    // shape groups run their GEMM chains concurrently on these (small groups
    // leave SMs idle; their persistent kernels overlap the big ones)
    static constexpr int kGroupStreams = 4;
    cudaStream_t gstream[kGroupStreams] = {};
    cudaEvent_t gfork = nullptr, gjoin[kGroupStreams] = {};
    cudaEvent_t ev_snap = nullptr;
    // scheduler
    double now_us = 0.0;
    std::mt19937_64 jitter;
    asg_pool_stats stats{};
    std::vector<asg_event> events;
    // refresh workspace (fp64), sized for a chunk of blocks of dim <= ws_n
    int ws_chunk = 0, ws_n = 0;
    double *ws_snap = nullptr, *ws_vecs = nullptr, *ws_work = nullptr, *ws_W = nullptr, *ws_out = nullptr,
           *ws_vals = nullptr, *ws_eps = nullptr;
    // F32 refresh workspace (side stream): 8 split-tf32 slabs of ws_chunk x D x D
    float* tw[8] = {};
    size_t tw_slab = 0;  // floats per block slot (Dmax^2)
    // F32 SOAP install workspace (main stream): 6 slabs of ws_chunk x D x D
    float* iw32[6] = {};
    // F32 refresh: tensor-core Jacobi workspace (side stream)
    float* tc_ws = nullptr;
    // NEWTON refresh: coupled Newton-Schulz workspace (side stream)
    float* ns_ws = nullptr;
    int* pair_status = nullptr;  // both-sides eigensolves: per-matrix status before the merge
    int* pair_ident = nullptr;   // both-sides eigensolves: per-matrix J = I flags
    // Refresh chunks alternate between two side streams, each with its own copy of the
    // side-stream workspace above (ws_* .. pair_ident): the active set is loaded into those
    // fields while a chunk's work is launched (kernels capture the pointers), set 0 otherwise.
    struct SideWs {
        double *snap, *vecs, *work, *W, *out, *vals, *eps;
        float* tw[8];
        float *tc_ws, *ns_ws;
        int *pair_status, *pair_ident;
    };
    SideWs side_ws[2] = {};
    int nside = 1;
    cudaStream_t side2 = nullptr;
    bool fp64_jacobi = false;  // ASG_F32_FP64_JACOBI=1: F32 refresh with the fp64 block Jacobi (diagnostics)
    // SOAP install workspace (one block)
    double *iw_rotL = nullptr, *iw_rotR = nullptr, *iw_sq = nullptr, *iw_a = nullptr, *iw_b = nullptr;
    // scalars
    int* d_flag = nullptr;      // gradient norm: non-finite gradient
    int* d_upd_flag = nullptr;  // update (EPI_APPLY, AdamW): non-finite update, surfaced at the next host sync
    int* h_upd_flag = nullptr;  // pinned copy, written on the main stream after every update
    // EVENT-mode barrier installs that did not block the host: the main stream
    // waits on the refresh event; the refresh status and the device-side wait
    // (ev_a -> ev_b on the main stream) are resolved at the next host sync
    struct DeferredInstall {
        int unit;
        cudaEvent_t ev_a, ev_b;
    };
    std::vector<DeferredInstall> deferred_status;
    double* d_sqnorm = nullptr;
    float* d_scale = nullptr;
    // parity staging
    float* stage = nullptr;
    size_t stage_elems = 0;
    asg::BlockRef* d_ref1 = nullptr;
    asg::ApplyEntry* d_apply1 = nullptr;
    float* d_out1 = nullptr;
    // multi-tensor gradient-norm chunks (every parameter)
    asg::SqChunk* d_sq = nullptr;
    int n_sq = 0;
    // multi-tensor AdamW table (owned 1-D / degenerate parameters)
    asg::AdamEntry* d_adam = nullptr;
    int n_adam = 0;
    int64_t adam_max_elems = 0;
    // multi-GPU pack layout
    asg::BlockRef* d_pack_refs = nullptr;
    int64_t* d_pack_offs = nullptr;
    int n_pack = 0;
    std::vector<int64_t> shard_elems;
    asg::BlockRef* d_unpack_refs = nullptr;
    int64_t* d_unpack_offs = nullptr;
    int n_unpack = 0;
    std::vector<int> unpack_rank;
    int64_t stride = 0;  // elements per rank segment of the owner-major buffers
    asg::BlockRef *d_gpack_refs = nullptr, *d_gunpack_refs = nullptr;
    int64_t *d_gpack_offs = nullptr, *d_gunpack_offs = nullptr;
    // bucketed parameter all-gather: buckets of each shape's
    // owned units, identical on every rank; with a communicator set, asg_step
    // all-gathers bucket b on comm_stream while the main stream updates b+1
    struct Bucket {
        bool adamw = false;
        int group = -1, s0 = 0, cnt = 0;  // this rank's slot range in its group for the shape
        int64_t stride = 0;                // elements per rank segment (the largest over ranks)
        asg::BlockRef *d_pack_refs = nullptr, *d_unpack_refs = nullptr;
        int64_t *d_pack_offs = nullptr, *d_unpack_offs = nullptr;
        int n_pack = 0, n_unpack = 0;
    };
    std::vector<Bucket> buckets;
    int buckets_per_shape = 0;
    void* ag_comm = nullptr;  // ncclComm_t (fused all-gather in asg_step)
    cudaStream_t comm_stream = nullptr;
    float *ag_send = nullptr, *ag_recv = nullptr;
    std::vector<cudaEvent_t> ag_events;
    cudaEvent_t ag_done = nullptr;
    // installs decided by the schedule bookkeeping, executed after the
    // step's refreshes are launched as one batch
    std::vector<int> deferred_installs;
    // profiling
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    struct HbmProf {
        cudaEvent_t e0, e1;
        int kind;
        double bytes;
    };
    std::vector<HbmProf> prof_hbm;  // HBM-bound kernels of the step (asg_hbm_stats kinds)
    double prof_flops = 0.0;
    uint64_t prof_gemms = 0;
    uint64_t launch_base = 0;
};

namespace asg {
namespace {

template <class T>
T* dalloc(asg_blockset* bs, size_t count) {
    if (count == 0) return nullptr;
    void* p = nullptr;
    CK(cudaMalloc(&p, count * sizeof(T)));
    bs->allocs.push_back(p);
    bs->alloc_bytes += count * sizeof(T);
    return static_cast<T*>(p);
}

template <class T>
T* halloc(asg_blockset* bs, size_t count) {
    void* p = nullptr;
    CK(cudaMallocHost(&p, std::max<size_t>(1, count) * sizeof(T)));
    bs->host_allocs.push_back(p);
    std::memset(p, 0, std::max<size_t>(1, count) * sizeof(T));
    return static_cast<T*>(p);
}

// H2D upload ordered on `s` and complete on return (a pageable cudaMemcpy may
// return before its DMA lands, and our streams do not sync with the legacy one).
void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
}

bool is_precond(const asg_blockset* bs) { return bs->opt.method != ASG_METHOD_ADAMW; }
bool is_soap(const asg_blockset* bs) { return bs->opt.method == ASG_METHOD_SOAP; }
bool is_kl(const asg_blockset* bs) { return bs->opt.method == ASG_METHOD_KL_SHAMPOO; }
// operand slabs of the state hold (hi, lo) pairs (3XTF32); 3XTF32_SMEM keeps
// them as plain fp32, split in shared memory by the GEMM (asg_gemm.cuh SPL)
bool split_mode(const asg_blockset* bs) { return bs->precision == ASG_PREC_3XTF32; }
// the refresh's internal tensor-core Jacobi works on (hi, lo) pairs in both 3xTF32 modes
bool work_split(const asg_blockset* bs) { return bs->precision != ASG_PREC_TF32; }
void to_f16(const float* src, int nb, int s0, int cnt, int64_t per, uint16_t* dst, float* scale, unsigned int* amax,
            cudaStream_t s, unsigned int* n1 = nullptr, int n = 0);
// 3XF16: the Shampoo / KL-Shampoo step chains on fp16 pairs (SOAP runs as 3XTF32_SMEM)
bool f16_mode(const asg_blockset* bs) {
    return bs->precision == ASG_PREC_3XF16 && bs->opt.method != ASG_METHOD_SOAP;
}
// F32 and NEWTON: fp32-level refresh (NEWTON: Newton-Schulz roots for Shampoo / KL)
bool f32_refresh(const asg_blockset* bs) { return bs->sc.refresh_mode != ASG_REFRESH_F64; }
bool newton_roots(const asg_blockset* bs) {
    return bs->sc.refresh_mode == ASG_REFRESH_NEWTON && bs->opt.method != ASG_METHOD_SOAP;
}
// Relative threshold of the F32 refresh's Jacobi (asg_eigh.cuh EighOpts).
constexpr double kF32RefreshTolDefault = 1e-6;
// ASG_F32_TOL overrides the threshold (diagnostics / tuning).
double f32_refresh_tol() {
    static const double t = getenv("ASG_F32_TOL") ? atof(getenv("ASG_F32_TOL")) : kF32RefreshTolDefault;
    return t;
}

void emit(asg_blockset* bs, int64_t step, int kind, int64_t block, uint64_t version, double t) {
    asg_event e{};
    e.step = step;
    e.kind = kind;
    e.block = block;
    e.version = version;
    e.t_us = t;
    bs->events.push_back(e);
}

size_t slabMM(const Group& g) { return size_t(g.M) * g.M; }
size_t slabNN(const Group& g) { return size_t(g.N) * g.N; }
size_t slabMN(const Group& g) { return size_t(g.M) * g.N; }

// ---------------------------------------------------------------------------
// construction
// ---------------------------------------------------------------------------
void build_units(asg_blockset* bs) {
    for (int64_t p = 0; p < int64_t(bs->params.size()); ++p) {
        const asg_param_desc& d = bs->params[size_t(p)];
        if (d.rows < 1 || d.cols < 1) throw Fail{ASG_ERR_SHAPE_MISMATCH, "partition_param: empty parameter"};
        const bool adamw = !is_precond(bs) || d.rows == 1 || d.cols == 1;  // harness.cpp:352
        if (adamw) {
            Unit u;
            u.spec = {p, 0, d.rows, 0, d.cols, bs->opt.block_dim_limit};
            u.adamw = true;
            u.cost = 28.0 * double(d.rows * d.cols) / 400.0;  // bytes -> flop-equivalent at ~400 flop/B
            bs->units.push_back(u);
            continue;
        }
        const int64_t limit = bs->opt.block_dim_limit;
        for (int64_t r = 0; r < d.rows; r += limit)  // partition_param precond.cpp:69-82
            for (int64_t c = 0; c < d.cols; c += limit) {
                Unit u;
                u.spec = {p, r, std::min(d.rows, r + limit), c, std::min(d.cols, c + limit), limit};
                const double m = double(u.spec.row_end - r), n = double(u.spec.col_end - c);
                const double step_w = (is_soap(bs) ? 5.0 : is_kl(bs) ? 5.0 : 3.0) * m * n * (m + n);
                const double refresh_w = 9.0 * (m * m * m + n * n * n);
                u.cost = step_w + refresh_w / double(bs->opt.precondition_frequency);
                bs->units.push_back(u);
            }
    }
    // LPT ownership: heaviest first onto the least-loaded rank.
    std::vector<int> order(bs->units.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = int(i);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return bs->units[size_t(a)].cost > bs->units[size_t(b)].cost; });
    std::vector<double> load(size_t(bs->world), 0.0);
    for (int i : order) {
        int best = 0;
        for (int r = 1; r < bs->world; ++r)
            if (load[size_t(r)] < load[size_t(best)]) best = r;
        bs->units[size_t(i)].owner = best;
        load[size_t(best)] += bs->units[size_t(i)].cost;
    }
}

void build_groups(asg_blockset* bs) {
    std::map<std::pair<int, int>, int> by_shape;
    for (size_t i = 0; i < bs->units.size(); ++i) {
        Unit& u = bs->units[i];
        if (u.adamw || u.owner != bs->rank) continue;
        const int m = int(u.spec.row_end - u.spec.row_begin), n = int(u.spec.col_end - u.spec.col_begin);
        auto key = std::make_pair(m, n);
        auto it = by_shape.find(key);
        if (it == by_shape.end()) {
            Group g;
            g.m = m;
            g.n = n;
            g.M = int(round_up(m, 128));
            g.N = int(round_up(n, 128));
            it = by_shape.emplace(key, int(bs->groups.size())).first;
            bs->groups.push_back(g);
        }
        Group& g = bs->groups[size_t(it->second)];
        u.group = it->second;
        u.slot = int(g.units.size());
        g.units.push_back(int(i));
    }
}

void bind_group_tables(asg_blockset* bs, Group& g) {
    std::vector<BlockRef> refs(size_t(g.nb));
    std::vector<ApplyEntry> app(size_t(g.nb));
    for (int s = 0; s < g.nb; ++s) {
        const Unit& u = bs->units[size_t(g.units[size_t(s)])];
        const asg_param_desc& d = bs->params[size_t(u.spec.param_index)];
        refs[size_t(s)].src = d.grad ? d.grad + u.spec.row_begin * d.ld_grad + u.spec.col_begin : nullptr;
        refs[size_t(s)].dst = nullptr;
        refs[size_t(s)].ld = d.ld_grad;
        refs[size_t(s)].rows = g.m;
        refs[size_t(s)].cols = g.n;
        app[size_t(s)].theta = d.theta ? d.theta + u.spec.row_begin * d.ld_theta + u.spec.col_begin : nullptr;
        app[size_t(s)].ld = d.ld_theta;
        app[size_t(s)].rows = g.m;
        app[size_t(s)].cols = g.n;
    }
    g.vec_grad = g.n % 4 == 0;
    for (int s2 = 0; s2 < g.nb; ++s2) {
        const Unit& u = bs->units[size_t(g.units[size_t(s2)])];
        const asg_param_desc& d = bs->params[size_t(u.spec.param_index)];
        const uintptr_t a = reinterpret_cast<uintptr_t>(refs[size_t(s2)].src);
        g.vec_grad = g.vec_grad && d.ld_grad % 4 == 0 && a % 16 == 0;
    }
    h2d(g.d_refs, refs.data(), refs.size() * sizeof(BlockRef), bs->main);
    h2d(g.d_apply, app.data(), app.size() * sizeof(ApplyEntry), bs->main);
}

void alloc_group(asg_blockset* bs, Group& g) {
    const bool sp = split_mode(bs);
    g.nb = int(g.units.size());
    const size_t nb = size_t(g.nb);
    g.L = dalloc<float>(bs, nb * slabMM(g));
    g.R = dalloc<float>(bs, nb * slabNN(g));
    // square blocks: the two sides' snapshots (and, below, roots) are one
    // allocation, so a refresh can batch both sides (refresh_newton)
    const bool joint = g.m == g.n;
    g.snapL = dalloc<float>(bs, (joint ? 2 : 1) * nb * slabMM(g));
    g.snapR = joint ? g.snapL + nb * slabMM(g) : dalloc<float>(bs, nb * slabNN(g));
    g.Gh = dalloc<float>(bs, nb * slabMN(g));
    g.GTh = dalloc<float>(bs, nb * slabMN(g));
    g.Th = dalloc<float>(bs, nb * slabMN(g));
    if (sp) {
        g.Gl = dalloc<float>(bs, nb * slabMN(g));
        g.GTl = dalloc<float>(bs, nb * slabMN(g));
        g.Tl = dalloc<float>(bs, nb * slabMN(g));
    }
    // S: SOAP's Adam output; KL-Shampoo's V^T, which aliases G (G is dead once
    // W = G P_R is formed; the update recomputes V from G^T, group_update);
    // Shampoo has no use for it
    if (is_soap(bs)) {
        g.Sh = dalloc<float>(bs, nb * slabMN(g));
        if (sp) g.Sl = dalloc<float>(bs, nb * slabMN(g));
    } else if (is_kl(bs)) {
        g.Sh = g.Gh;
        g.Sl = g.Gl;
    }
    if (f16_mode(bs)) {
        g.G16 = reinterpret_cast<uint16_t*>(g.Gh);  // prep writes fp16 pairs; no fp32 G in this mode
        g.GT16 = reinterpret_cast<uint16_t*>(g.GTh);
        // the step's products are written as fp16 pairs straight from the GEMM epilogue, so
        // the fp32 T slab holds T16; KL's V^T pairs (S16) alias G16, dead once W = G P_R is formed
        g.T16 = reinterpret_cast<uint16_t*>(g.Th);
        if (is_kl(bs)) g.S16 = g.G16;
        g.PL16 = reinterpret_cast<uint16_t*>(dalloc<float>(bs, nb * slabMM(g)));
        g.PR16 = reinterpret_cast<uint16_t*>(dalloc<float>(bs, nb * slabNN(g)));
        for (float** sc : {&g.gscale, &g.tscale, &g.sscale, &g.plscale, &g.prscale}) *sc = dalloc<float>(bs, nb);
        g.amax = dalloc<unsigned int>(bs, nb);
        g.amax2 = dalloc<unsigned int>(bs, nb);
        g.pln1 = dalloc<unsigned int>(bs, nb);
        g.prn1 = dalloc<unsigned int>(bs, nb);
        g.amaxp = dalloc<unsigned int>(bs, nb);
        g.gfix = dalloc<int>(bs, nb);
        CK(cudaMemsetAsync(g.amaxp, 0, nb * sizeof(unsigned int), bs->main));
    }
    auto pair_mm = [&](float*& h, float*& l) {
        h = dalloc<float>(bs, nb * slabMM(g));
        if (sp) l = dalloc<float>(bs, nb * slabMM(g));
    };
    auto pair_nn = [&](float*& h, float*& l) {
        h = dalloc<float>(bs, nb * slabNN(g));
        if (sp) l = dalloc<float>(bs, nb * slabNN(g));
    };
    cudaStream_t s = bs->main;
    if (is_soap(bs)) {
        pair_mm(g.QLh, g.QLl);
        pair_mm(g.QLTh, g.QLTl);
        pair_nn(g.QRh, g.QRl);
        pair_nn(g.QRTh, g.QRTl);
        g.mom_m = dalloc<float>(bs, nb * slabMN(g));
        g.mom_v = dalloc<float>(bs, nb * slabMN(g));
        if (f32_refresh(bs)) {
            pair_mm(g.sJLTh, g.sJLTl);
            pair_nn(g.sJRTh, g.sJRTl);
        } else {
            g.QL64 = dalloc<double>(bs, nb * size_t(g.m) * g.m);
            g.QR64 = dalloc<double>(bs, nb * size_t(g.n) * g.n);
            g.sQL64 = dalloc<double>(bs, nb * size_t(g.m) * g.m);
            g.sQR64 = dalloc<double>(bs, nb * size_t(g.n) * g.n);
        }
        g.valsL = dalloc<double>(bs, nb * size_t(g.m));
        g.valsR = dalloc<double>(bs, nb * size_t(g.n));
        g.svalsL = dalloc<double>(bs, nb * size_t(g.m));
        g.svalsR = dalloc<double>(bs, nb * size_t(g.n));
        launch_identity_split(g.QLh, g.QLl, g.nb, g.M, g.m, s);
        launch_identity_split(g.QLTh, g.QLTl, g.nb, g.M, g.m, s);
        launch_identity_split(g.QRh, g.QRl, g.nb, g.N, g.n, s);
        launch_identity_split(g.QRTh, g.QRTl, g.nb, g.N, g.n, s);
        // fp64 identity bases, eigenvalues 1 (EigenPair::identity densela.hpp:119-121)
        std::vector<double> eyeL(size_t(g.m) * g.m, 0.0), eyeR(size_t(g.n) * g.n, 0.0);
        for (int i = 0; i < g.m; ++i) eyeL[size_t(i) * g.m + i] = 1.0;
        for (int i = 0; i < g.n; ++i) eyeR[size_t(i) * g.n + i] = 1.0;
        std::vector<double> onesL(size_t(g.m), 1.0), onesR(size_t(g.n), 1.0);
        for (size_t b = 0; b < nb; ++b) {
            if (g.QL64) h2d(g.QL64 + b * g.m * g.m, eyeL.data(), eyeL.size() * 8, bs->main);
            if (g.QR64) h2d(g.QR64 + b * g.n * g.n, eyeR.data(), eyeR.size() * 8, bs->main);
            h2d(g.valsL + b * g.m, onesL.data(), onesL.size() * 8, bs->main);
            h2d(g.valsR + b * g.n, onesR.data(), onesR.size() * 8, bs->main);
        }
        CK(cudaMemsetAsync(g.mom_m, 0, nb * slabMN(g) * 4, s));
        CK(cudaMemsetAsync(g.mom_v, 0, nb * slabMN(g) * 4, s));
    } else {
        // joint (square) allocation of a left/right pair: R follows L
        auto pair_lr = [&](float*& lh, float*& ll, float*& rh, float*& rl) {
            if (!joint) {
                pair_mm(lh, ll);
                pair_nn(rh, rl);
                return;
            }
            lh = dalloc<float>(bs, 2 * nb * slabMM(g));
            rh = lh + nb * slabMM(g);
            if (sp) {
                ll = dalloc<float>(bs, 2 * nb * slabMM(g));
                rl = ll + nb * slabMM(g);
            }
        };
        pair_mm(g.PLh, g.PLl);
        pair_nn(g.PRh, g.PRl);
        pair_lr(g.sPLh, g.sPLl, g.sPRh, g.sPRl);
        launch_identity_split(g.PLh, g.PLl, g.nb, g.M, g.m, s);
        launch_identity_split(g.PRh, g.PRl, g.nb, g.N, g.n, s);
        if (f16_mode(bs)) {
            to_f16(g.PLh, g.nb, 0, g.nb, int64_t(slabMM(g)), g.PL16, g.plscale, g.amax, s, g.pln1, g.M);
            to_f16(g.PRh, g.nb, 0, g.nb, int64_t(slabNN(g)), g.PR16, g.prscale, g.amax, s, g.prn1, g.N);
        }
        if (f32_refresh(bs) && !newton_roots(bs)) {  // basis of the last refresh, identity before the first
            pair_mm(g.BLh, g.BLl);
            pair_mm(g.BLTh, g.BLTl);
            pair_nn(g.BRh, g.BRl);
            pair_nn(g.BRTh, g.BRTl);
            launch_identity_split(g.BLh, g.BLl, g.nb, g.M, g.m, s);
            launch_identity_split(g.BLTh, g.BLTl, g.nb, g.M, g.m, s);
            launch_identity_split(g.BRh, g.BRl, g.nb, g.N, g.n, s);
            launch_identity_split(g.BRTh, g.BRTl, g.nb, g.N, g.n, s);
        } else if (!f32_refresh(bs)) {
            g.EL64 = dalloc<double>(bs, nb * size_t(g.m) * g.m);
            g.ER64 = dalloc<double>(bs, nb * size_t(g.n) * g.n);
        }
        g.v_ok.assign(nb, 0);
    }
    // statistics: zero (precond.cpp:89-90); KL-Shampoo starts from identity
    launch_identity_f32(g.L, g.nb, g.M, g.m, is_kl(bs) ? 1.f : 0.f, s);
    launch_identity_f32(g.R, g.nb, g.N, g.n, is_kl(bs) ? 1.f : 0.f, s);
    CK(cudaMemsetAsync(g.Gh, 0, nb * slabMN(g) * 4, s));
    CK(cudaMemsetAsync(g.GTh, 0, nb * slabMN(g) * 4, s));
    if (sp) {
        CK(cudaMemsetAsync(g.Gl, 0, nb * slabMN(g) * 4, s));
        CK(cudaMemsetAsync(g.GTl, 0, nb * slabMN(g) * 4, s));
    }
    g.d_refs = dalloc<BlockRef>(bs, nb);
    g.d_apply = dalloc<ApplyEntry>(bs, nb);
    g.d_status = dalloc<int>(bs, nb);
    g.h_status = halloc<int>(bs, nb);
    if (f32_refresh(bs) && is_soap(bs)) {
        g.d_identL = dalloc<int>(bs, nb);
        g.d_identR = dalloc<int>(bs, nb);
        g.h_identL = halloc<int>(bs, nb);
        g.h_identR = halloc<int>(bs, nb);
        CK(cudaMemsetAsync(g.d_identL, 0, nb * sizeof(int), s));
        CK(cudaMemsetAsync(g.d_identR, 0, nb * sizeof(int), s));
    }
    CK(cudaMemsetAsync(g.d_status, 0, nb * sizeof(int), s));
    const int bnM = gemm_bn_for(g.M, nb), bnN = gemm_bn_for(g.N, nb);
    g.ntM = gemm_sym_tile_list(g.M, bnM, nullptr);
    g.ntN = gemm_sym_tile_list(g.N, bnN, nullptr);
    std::vector<int2> tl(size_t(std::max(g.ntM, g.ntN)));
    g.tilesM = dalloc<int2>(bs, size_t(g.ntM));
    gemm_sym_tile_list(g.M, bnM, tl.data());
    h2d(g.tilesM, tl.data(), size_t(g.ntM) * sizeof(int2), bs->main);
    g.tilesN = dalloc<int2>(bs, size_t(g.ntN));
    gemm_sym_tile_list(g.N, bnN, tl.data());
    h2d(g.tilesN, tl.data(), size_t(g.ntN) * sizeof(int2), bs->main);
    bind_group_tables(bs, g);
}

asg_blockset::SideWs save_side_ws(const asg_blockset* bs) {
    asg_blockset::SideWs w{};
    w.snap = bs->ws_snap;
    w.vecs = bs->ws_vecs;
    w.work = bs->ws_work;
    w.W = bs->ws_W;
    w.out = bs->ws_out;
    w.vals = bs->ws_vals;
    w.eps = bs->ws_eps;
    for (int k = 0; k < 8; ++k) w.tw[k] = bs->tw[k];
    w.tc_ws = bs->tc_ws;
    w.ns_ws = bs->ns_ws;
    w.pair_status = bs->pair_status;
    w.pair_ident = bs->pair_ident;
    return w;
}
void load_side_ws(asg_blockset* bs, const asg_blockset::SideWs& w) {
    bs->ws_snap = w.snap;
    bs->ws_vecs = w.vecs;
    bs->ws_work = w.work;
    bs->ws_W = w.W;
    bs->ws_out = w.out;
    bs->ws_vals = w.vals;
    bs->ws_eps = w.eps;
    for (int k = 0; k < 8; ++k) bs->tw[k] = w.tw[k];
    bs->tc_ws = w.tc_ws;
    bs->ns_ws = w.ns_ws;
    bs->pair_status = w.pair_status;
    bs->pair_ident = w.pair_ident;
}
void sync_side(asg_blockset* bs) {
    if (bs->side) CK(cudaStreamSynchronize(bs->side));
    if (bs->side2) CK(cudaStreamSynchronize(bs->side2));
}

void alloc_workspace(asg_blockset* bs) {
    int nmax = 0;
    size_t state_per_block = 0;
    for (const Group& g : bs->groups) {
        nmax = std::max({nmax, g.m, g.n});
        state_per_block = std::max(state_per_block, size_t(g.m) * g.m + size_t(g.n) * g.n);
    }
    if (nmax == 0) return;
    // Chunk the refresh so its fp64 workspace stays ~<= 4 GiB.
    const size_t per = size_t(nmax) * nmax * 8 * 7;
    int chunk = int(std::max<size_t>(1, (size_t(4) << 30) / per));
    int maxnb = 0;
    for (const Group& g : bs->groups) maxnb = std::max(maxnb, g.nb);
    bs->ws_chunk = std::min(chunk, std::max(1, maxnb));
    bs->ws_n = nmax;
    // NEWTON refresh: the fp64 buffers only stage single-block parity I/O
    // (asg_block_read / asg_block_write), so they hold one block, not a chunk
    auto alloc_side = [&]() {
        const size_t nn = size_t(nmax) * nmax * size_t(newton_roots(bs) ? 1 : bs->ws_chunk);
        bs->ws_snap = dalloc<double>(bs, nn);
        bs->ws_vecs = dalloc<double>(bs, nn);
        size_t ew = nn;
        if (!newton_roots(bs)) {
            for (const Group& g : bs->groups) {
                ew = std::max(ew, eigh_workspace_doubles(bs->ws_chunk, g.m));
                ew = std::max(ew, eigh_workspace_doubles(bs->ws_chunk, g.n));
            }
            for (const Group& g : bs->groups) {
                ew = std::max(ew, eigh_workspace_doubles_warm(bs->ws_chunk, g.m));
                ew = std::max(ew, eigh_workspace_doubles_warm(bs->ws_chunk, g.n));
            }
        }
        bs->ws_work = dalloc<double>(bs, ew);
        bs->ws_W = dalloc<double>(bs, nn);
        bs->ws_out = dalloc<double>(bs, nn);
        bs->ws_vals = dalloc<double>(bs, size_t(nmax) * bs->ws_chunk * 2);
        bs->ws_eps = dalloc<double>(bs, size_t(bs->ws_chunk) * 2);
        if (newton_roots(bs)) {
            int Dmax = 0;
            for (const Group& g : bs->groups) Dmax = std::max({Dmax, g.M, g.N});
            // both sides of a small square group run as one batch (refresh_newton)
            bool both = false;
            for (const Group& g : bs->groups) both |= g.m == g.n && g.nb <= bs->ws_chunk;
            bs->ns_ws = dalloc<float>(bs, ns_workspace_floats((both ? 2 : 1) * bs->ws_chunk, Dmax));
            bs->pair_status = dalloc<int>(bs, size_t(2 * bs->ws_chunk));
        } else if (f32_refresh(bs)) {
            int Dmax = 0;
            for (const Group& g : bs->groups) Dmax = std::max({Dmax, g.M, g.N});
            bs->tw_slab = size_t(Dmax) * Dmax;
            // two factor sides per chunk (square blocks share one eigensolve)
            for (float*& t : bs->tw) t = dalloc<float>(bs, bs->tw_slab * size_t(2 * bs->ws_chunk));
            bs->tc_ws = dalloc<float>(bs, tc_eigh_workspace_floats(2 * bs->ws_chunk, Dmax));
            bs->pair_status = dalloc<int>(bs, size_t(2 * bs->ws_chunk));
            bs->pair_ident = dalloc<int>(bs, size_t(2 * bs->ws_chunk));
        }
    };
    alloc_side();
    bs->side_ws[0] = save_side_ws(bs);
    // a second set for the second refresh stream when a dispatch can launch more than one
    // chunk (several shape groups, or a group larger than a chunk); ASG_REFRESH_STREAMS=1: one
    int maxnb2 = 0;
    for (const Group& g : bs->groups) maxnb2 = std::max(maxnb2, g.nb);
    static const int want = getenv("ASG_REFRESH_STREAMS") ? atoi(getenv("ASG_REFRESH_STREAMS")) : 2;
    if (want >= 2 && (bs->groups.size() > 1 || maxnb2 > bs->ws_chunk)) {
        alloc_side();
        bs->side_ws[1] = save_side_ws(bs);
        bs->nside = 2;
        load_side_ws(bs, bs->side_ws[0]);
    }
    if (f32_refresh(bs) && !newton_roots(bs) && is_soap(bs))
        for (float*& t : bs->iw32) t = dalloc<float>(bs, bs->tw_slab * size_t(bs->ws_chunk));
    if (is_soap(bs)) {
        int maxmn = 0;
        for (const Group& g : bs->groups) maxmn = std::max(maxmn, g.m * g.n);
        bs->iw_rotL = dalloc<double>(bs, size_t(nmax) * nmax);
        bs->iw_rotR = dalloc<double>(bs, size_t(nmax) * nmax);
        bs->iw_sq = dalloc<double>(bs, size_t(nmax) * nmax);
        bs->iw_a = dalloc<double>(bs, size_t(maxmn));
        bs->iw_b = dalloc<double>(bs, size_t(maxmn));
    }
}

// ---------------------------------------------------------------------------
// GEMM helpers
// ---------------------------------------------------------------------------
Operand op(const float* h, const float* l, int rows, int K) { return Operand{h, l, rows, K}; }
// slots [s0, ...) of an fp16-pair slab of nb blocks of rows x K, with their scales
Operand op16(const uint16_t* base, int nb, int s0, int rows, int K, const float* scale) {
    const size_t per = size_t(rows) * K;
    return Operand{reinterpret_cast<const float*>(base + size_t(s0) * per),
                   reinterpret_cast<const float*>(base + size_t(nb) * per + size_t(s0) * per), rows, K, scale + s0};
}
// fp32 slots [s0, s0+cnt) (rows x K each) -> fp16 pairs + scales of the same slots
void to_f16(const float* src, int nb, int s0, int cnt, int64_t per, uint16_t* dst, float* scale, unsigned int* amax,
            cudaStream_t s, unsigned int* n1, int n) {
    launch_absmax(src + size_t(s0) * per, cnt, per, amax + s0, s);
    // a root's 1-norm bounds the products it enters (|G P|_ij <= max|G| |P|_1): the fp16
    // scale of those products is fixed before them, so they write fp16 pairs directly
    if (n1) launch_colabs_max(src + size_t(s0) * per, cnt, n, per, n1 + s0, s);
    launch_to_f16pair(src + size_t(s0) * per, amax + s0, cnt, per, dst + size_t(s0) * per,
                      dst + size_t(nb) * per + size_t(s0) * per, scale + s0, s);
}

void run_gemm(asg_blockset* bs, Operand A, Operand B, int batch, int epi, const GemmParams& p,
              const int2* sym_tiles, int nsym, cudaStream_t s, double alg_flops) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    // profile the step's GEMMs (main and group streams); refresh GEMMs on the
    // side stream overlap them and are not part of the step's roofline
    if (bs->profiling && s != bs->side && s != bs->side2) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, s));
    }
    GemmLaunch g{};
    g.A = A;
    g.B = B;
    g.batch = batch;
    g.epi = epi;
    g.p = p;
    g.sym_tiles = sym_tiles;
    g.sym_tiles_count = nsym;
    CK(gemm_launch(g, bs->precision, bs->num_sms, s));
    if (e0) {
        CK(cudaEventRecord(e1, s));
        bs->prof_events.emplace_back(e0, e1);
        bs->prof_flops += alg_flops;
        bs->prof_gemms += 1;
    }
}

// Brackets an HBM-bound launch with CUDA events on its stream while profiling
// (asg_get_hbm_stats): kind, algorithmic bytes.
template <class F>
void hbm_launch(asg_blockset* bs, cudaStream_t s, int kind, double bytes, F&& launch) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (bs->profiling) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, s));
    }
    launch();
    if (e0) {
        CK(cudaEventRecord(e1, s));
        bs->prof_hbm.push_back({e0, e1, kind, bytes});
    }
}

template <class T>
T* at(T* base, size_t stride, int slot) {
    return base ? base + stride * size_t(slot) : nullptr;
}

// (Re)builds the owner-major layouts of the multi-GPU exchange:
// rank r's owned units are contiguous at r * stride (stride = the largest shard):
//   theta pack (owned) / theta unpack (all units, after the all-gather),
//   gradient pack (all units, before a reduce-scatter) / gradient unpack (owned).
void build_owner_layout(asg_blockset* bs) {
    std::vector<BlockRef> pk, upk, gpk, gupk;
    std::vector<int64_t> pko, upko, gpko, gupko;
    std::vector<int64_t> inrank;
    bs->shard_elems.assign(size_t(bs->world), 0);
    bs->unpack_rank.clear();
    for (int r = 0; r < bs->world; ++r)
        for (size_t i = 0; i < bs->units.size(); ++i) {
            const Unit& u = bs->units[i];
            if (u.owner != r) continue;
            const asg_param_desc& d = bs->params[size_t(u.spec.param_index)];
            const int32_t rows = int32_t(u.spec.row_end - u.spec.row_begin), cols = int32_t(u.spec.col_end - u.spec.col_begin);
            BlockRef th{}, gr{};
            th.src = th.dst = d.theta ? d.theta + u.spec.row_begin * d.ld_theta + u.spec.col_begin : nullptr;
            th.ld = d.ld_theta;
            th.rows = rows;
            th.cols = cols;
            gr.src = d.grad ? d.grad + u.spec.row_begin * d.ld_grad + u.spec.col_begin : nullptr;
            gr.dst = const_cast<float*>(gr.src);
            gr.ld = d.ld_grad;
            gr.rows = rows;
            gr.cols = cols;
            const int64_t at_rank = bs->shard_elems[size_t(r)];
            if (r == bs->rank) {
                pk.push_back(th);
                pko.push_back(at_rank);
                gupk.push_back(gr);
                gupko.push_back(at_rank);
            }
            upk.push_back(th);
            gpk.push_back(gr);
            inrank.push_back(at_rank);
            bs->unpack_rank.push_back(r);
            bs->shard_elems[size_t(r)] += int64_t(rows) * cols;
        }
    bs->stride = 0;
    for (int64_t e : bs->shard_elems) bs->stride = std::max(bs->stride, e);
    for (size_t i = 0; i < upk.size(); ++i) {
        upko.push_back(int64_t(bs->unpack_rank[i]) * bs->stride + inrank[i]);
        gpko.push_back(int64_t(bs->unpack_rank[i]) * bs->stride + inrank[i]);
    }
    bs->n_pack = int(pk.size());
    bs->n_unpack = int(upk.size());
    auto up = [&](auto*& dst, const auto& v) {
        using T = typename std::decay_t<decltype(v)>::value_type;
        if (!dst) dst = dalloc<T>(bs, std::max<size_t>(1, bs->units.size()));
        if (!v.empty()) h2d(dst, v.data(), v.size() * sizeof(T), bs->main);
    };
    up(bs->d_pack_refs, pk);
    up(bs->d_pack_offs, pko);
    up(bs->d_unpack_refs, upk);
    up(bs->d_unpack_offs, upko);
    up(bs->d_gpack_refs, gpk);
    up(bs->d_gpack_offs, gpko);
    up(bs->d_gunpack_refs, gupk);
    up(bs->d_gunpack_offs, gupko);
}

// Buckets of the parameter all-gather. For each block shape (in order of
// first appearance among all units; 1-D AdamW parameters last share one
// key), every rank's units of that shape in unit order are split into
// `per_shape` runs of B = ceil(max_r n_r / per_shape) units; bucket (shape, c)
// holds run c of every rank. The plan is a pure function of the ownership
// plan, so every rank builds the same bucket list and issues the same
// collectives. A rank's run c of a shape is slots [cB, cB + cnt) of its group
// (slots follow unit order, build_groups).
void build_buckets(asg_blockset* bs, int per_shape) {
    for (auto& b : bs->buckets)
        for (void* p : {static_cast<void*>(b.d_pack_refs), static_cast<void*>(b.d_unpack_refs),
                        static_cast<void*>(b.d_pack_offs), static_cast<void*>(b.d_unpack_offs)})
            if (p) {
                cudaFree(p);
                bs->allocs.erase(std::remove(bs->allocs.begin(), bs->allocs.end(), p), bs->allocs.end());
            }
    bs->buckets.clear();
    bs->buckets_per_shape = per_shape;
    std::vector<std::pair<int, int>> keys;
    std::map<std::pair<int, int>, std::vector<std::vector<int>>> lists;  // key -> rank -> units
    for (size_t i = 0; i < bs->units.size(); ++i) {
        const Unit& u = bs->units[i];
        const std::pair<int, int> key =
            u.adamw ? std::make_pair(-1, -1)
                    : std::make_pair(int(u.spec.row_end - u.spec.row_begin), int(u.spec.col_end - u.spec.col_begin));
        auto it = lists.find(key);
        if (it == lists.end()) {
            it = lists.emplace(key, std::vector<std::vector<int>>(size_t(bs->world))).first;
            if (key.first >= 0) keys.push_back(key);
        }
        it->second[size_t(u.owner)].push_back(int(i));
    }
    if (lists.count({-1, -1})) keys.push_back({-1, -1});
    auto slice = [&](const Unit& u) {
        const asg_param_desc& d = bs->params[size_t(u.spec.param_index)];
        BlockRef th{};
        th.src = th.dst = d.theta ? d.theta + u.spec.row_begin * d.ld_theta + u.spec.col_begin : nullptr;
        th.ld = d.ld_theta;
        th.rows = int32_t(u.spec.row_end - u.spec.row_begin);
        th.cols = int32_t(u.spec.col_end - u.spec.col_begin);
        return th;
    };
    for (const auto& key : keys) {
        const auto& per_rank = lists[key];
        size_t nmax = 0;
        for (const auto& l : per_rank) nmax = std::max(nmax, l.size());
        if (nmax == 0) continue;
        const size_t B = key.first < 0 ? nmax : (nmax + size_t(per_shape) - 1) / size_t(per_shape);
        int my_group = -1;
        for (size_t gi = 0; gi < bs->groups.size(); ++gi)
            if (bs->groups[gi].m == key.first && bs->groups[gi].n == key.second) my_group = int(gi);
        for (size_t c0 = 0; c0 < nmax; c0 += B) {
            asg_blockset::Bucket bk;
            bk.adamw = key.first < 0;
            std::vector<int64_t> elems(size_t(bs->world), 0);
            for (int r = 0; r < bs->world; ++r)
                for (size_t j = c0; j < std::min(c0 + B, per_rank[size_t(r)].size()); ++j) {
                    const Unit& u = bs->units[size_t(per_rank[size_t(r)][j])];
                    elems[size_t(r)] += (u.spec.row_end - u.spec.row_begin) * (u.spec.col_end - u.spec.col_begin);
                }
            for (int64_t e : elems) bk.stride = std::max(bk.stride, e);
            const auto& mine = per_rank[size_t(bs->rank)];
            bk.group = bk.adamw ? -1 : my_group;
            bk.s0 = int(c0);
            bk.cnt = int(std::min(c0 + B, mine.size()) > c0 ? std::min(c0 + B, mine.size()) - c0 : 0);
            std::vector<BlockRef> pk, upk;
            std::vector<int64_t> pko, upko;
            int64_t off = 0;
            for (size_t j = c0; j < std::min(c0 + B, mine.size()); ++j) {
                const Unit& u = bs->units[size_t(mine[j])];
                pk.push_back(slice(u));
                pko.push_back(off);
                off += int64_t(pk.back().rows) * pk.back().cols;
            }
            for (int r = 0; r < bs->world; ++r) {
                int64_t o = int64_t(r) * bk.stride;
                for (size_t j = c0; j < std::min(c0 + B, per_rank[size_t(r)].size()); ++j) {
                    const Unit& u = bs->units[size_t(per_rank[size_t(r)][j])];
                    upk.push_back(slice(u));
                    upko.push_back(o);
                    o += int64_t(upk.back().rows) * upk.back().cols;
                }
            }
            bk.n_pack = int(pk.size());
            bk.n_unpack = int(upk.size());
            if (!pk.empty()) {
                bk.d_pack_refs = dalloc<BlockRef>(bs, pk.size());
                bk.d_pack_offs = dalloc<int64_t>(bs, pko.size());
                h2d(bk.d_pack_refs, pk.data(), pk.size() * sizeof(BlockRef), bs->main);
                h2d(bk.d_pack_offs, pko.data(), pko.size() * sizeof(int64_t), bs->main);
            }
            if (!upk.empty()) {
                bk.d_unpack_refs = dalloc<BlockRef>(bs, upk.size());
                bk.d_unpack_offs = dalloc<int64_t>(bs, upko.size());
                h2d(bk.d_unpack_refs, upk.data(), upk.size() * sizeof(BlockRef), bs->main);
                h2d(bk.d_unpack_offs, upko.data(), upko.size() * sizeof(int64_t), bs->main);
            }
            bs->buckets.push_back(bk);
        }
    }
    int64_t smax = 0;
    for (const auto& b : bs->buckets) smax = std::max(smax, b.stride);
    for (float* p : {bs->ag_send, bs->ag_recv})
        if (p) {
            cudaFree(p);
            bs->allocs.erase(std::remove(bs->allocs.begin(), bs->allocs.end(), static_cast<void*>(p)), bs->allocs.end());
        }
    bs->ag_send = dalloc<float>(bs, size_t(std::max<int64_t>(1, smax)));
    bs->ag_recv = dalloc<float>(bs, size_t(std::max<int64_t>(1, smax)) * size_t(bs->world));
}

// NCCL, loaded at run time (libnccl.so.2: the copy torch already mapped, or
// the system one), so the library links without it and fails loudly only when
// a collective is requested.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};
const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.GetErrorString;
        return a;
    }();
    if (!api.ok) throw Fail{ASG_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) not loadable"};
    return api;
}
void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Fail{ASG_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r)};
}

// Bucket b: pack this rank's updated slices, all-gather, scatter every rank's
// slices into the parameters (all on stream s).
void bucket_exchange(asg_blockset* bs, const asg_blockset::Bucket& b, ncclComm_t comm, cudaStream_t s) {
    launch_pack_blocks(b.d_pack_refs, b.d_pack_offs, b.n_pack, bs->ag_send, s);
    nccl_check(nccl().AllGather(bs->ag_send, bs->ag_recv, size_t(b.stride), ncclFloat32, comm, s), "ncclAllGather");
    launch_unpack_blocks(b.d_unpack_refs, b.d_unpack_offs, b.n_unpack, bs->ag_recv, s);
}

// (Re)builds the chunk table of the one-launch global gradient norm.
void build_sq_table(asg_blockset* bs) {
    // chunks of 2^12..2^16 elements (multiples of 1024, so every chunk of a
    // contiguous gradient keeps 16-byte loads), at least ~4 CTAs per SM when the
    // gradients are small (one 1024^2 block: 16 chunks of 2^16 took 23 us)
    int64_t total = 0;
    for (const asg_param_desc& d : bs->params)
        if (d.grad) total += d.rows * d.cols;
    const int64_t want = (total / (4 * int64_t(bs->num_sms)) + 1023) / 1024 * 1024;
    const int64_t kChunkElems = std::max<int64_t>(4096, std::min<int64_t>(int64_t(1) << 16, want));
    std::vector<SqChunk> t;
    for (const asg_param_desc& d : bs->params) {
        if (!d.grad) continue;
        const int64_t n = d.rows * d.cols;
        for (int64_t e = 0; e < n; e += kChunkElems) t.push_back({d.grad, d.ld_grad, d.cols, e, std::min(n, e + kChunkElems)});
    }
    if (bs->d_sq && int(t.size()) > bs->n_sq) throw Fail{ASG_ERR_SHAPE_MISMATCH, "gradient chunk table grew"};
    bs->n_sq = int(t.size());
    if (t.empty()) return;
    if (!bs->d_sq) bs->d_sq = dalloc<SqChunk>(bs, t.size());
    h2d(bs->d_sq, t.data(), t.size() * sizeof(SqChunk), bs->main);
}

// (Re)builds the device table of the multi-tensor AdamW launch.
void build_adam_table(asg_blockset* bs) {
    std::vector<AdamEntry> t;
    bs->adam_max_elems = 0;
    for (const Unit& u : bs->units) {
        if (!u.adamw || u.owner != bs->rank) continue;
        const asg_param_desc& d = bs->params[size_t(u.spec.param_index)];
        AdamEntry e{d.theta, d.grad, u.am, u.av, d.ld_theta, d.ld_grad, d.rows, d.cols};
        t.push_back(e);
        bs->adam_max_elems = std::max(bs->adam_max_elems, d.rows * d.cols);
    }
    bs->n_adam = int(t.size());
    if (t.empty()) return;
    if (!bs->d_adam) bs->d_adam = dalloc<AdamEntry>(bs, t.size());
    h2d(bs->d_adam, t.data(), t.size() * sizeof(AdamEntry), bs->main);
}

// Concurrent group chains: fork from the main stream, run group i on
// stream_for(i), join back. With one group everything stays on main.
int fork_groups(asg_blockset* bs) {
    // Off by default: measured no gain on C2 (the step's big groups already fill
    // the GPU), and overlapping launches would blur the per-GEMM timing of
    // the roofline. ASG_GROUP_STREAMS=1 enables it.
    static const bool on = getenv("ASG_GROUP_STREAMS") != nullptr;
    if (!on) return 0;
    const int k = std::min<int>(asg_blockset::kGroupStreams, int(bs->groups.size()));
    if (k <= 1) return 0;
    CK(cudaEventRecord(bs->gfork, bs->main));
    for (int i = 0; i < k; ++i) CK(cudaStreamWaitEvent(bs->gstream[i], bs->gfork, 0));
    return k;
}
cudaStream_t stream_for(asg_blockset* bs, int k, int i) { return k ? bs->gstream[i % k] : bs->main; }
void join_groups(asg_blockset* bs, int k) {
    for (int i = 0; i < k; ++i) {
        CK(cudaEventRecord(bs->gjoin[i], bs->gstream[i]));
        CK(cudaStreamWaitEvent(bs->main, bs->gjoin[i], 0));
    }
}

// Statistics for slots [s0, s0+cnt) of a group (G slabs already staged).
// 3XF16 statistics (same products as group_stats; operands fp16 pairs with
// per-block scales; every fp32 intermediate is converted once, to_f16).
void group_stats_f16(asg_blockset* bs, Group& g, int s0, int cnt, cudaStream_t s) {
    const asg_optimizer_config& o = bs->opt;
    const double mf = g.m, nf = g.n;
    const bool ema = o.accumulation == ASG_ACCUM_EMA;
    const size_t mn = slabMN(g), mm = slabMM(g), nn = slabNN(g);
    const int nb = g.nb;
    GemmParams p{};
    p.beta = ema ? float(o.beta2) : 1.f;
    if (!is_kl(bs)) {
        p.alpha = ema ? float(1.0 - o.beta2) : 1.f;
        p.C = at(g.L, mm, s0);
        p.ldc = g.M;
        p.c_bstride = int64_t(mm);
        const Operand gop = op16(g.G16, nb, s0, g.M, g.N, g.gscale);
        run_gemm(bs, gop, gop, cnt, EPI_SYM_EMA, p, g.tilesM, g.ntM, s, cnt * mf * mf * nf);
        p.C = at(g.R, nn, s0);
        p.ldc = g.N;
        p.c_bstride = int64_t(nn);
        const Operand gtop = op16(g.GT16, nb, s0, g.N, g.M, g.gscale);
        run_gemm(bs, gtop, gtop, cnt, EPI_SYM_EMA, p, g.tilesN, g.ntN, s, cnt * nf * nf * mf);
        return;
    }
    // W = G P_R -> T16 (fp16 pairs at the scale of the bound max|G| |P_R|_1) ; L = b L + a/n W W^T
    GemmParams px{};
    px.alpha = 1.f;
    px.ldd = g.N;
    px.d_bstride = int64_t(mn);
    launch_bound_scale(cnt, g.gscale + s0, g.prn1 + s0, g.tscale + s0, nullptr, s);
    px.Dhi = reinterpret_cast<float*>(g.T16 + size_t(s0) * mn);
    px.Dlo = reinterpret_cast<float*>(g.T16 + size_t(nb) * mn + size_t(s0) * mn);
    px.oscale = g.tscale + s0;
    run_gemm(bs, op16(g.G16, nb, s0, g.M, g.N, g.gscale), op16(g.PR16, nb, s0, g.N, g.N, g.prscale), cnt, EPI_SPLIT,
             px, nullptr, 0, s, cnt * 2.0 * mf * nf * nf);
    const double a = ema ? (1.0 - o.beta2) : 1.0;
    p.alpha = float(a / double(g.n));
    p.C = at(g.L, mm, s0);
    p.ldc = g.M;
    p.c_bstride = int64_t(mm);
    const Operand wop = op16(g.T16, nb, s0, g.M, g.N, g.tscale);
    run_gemm(bs, wop, wop, cnt, EPI_SYM_EMA, p, g.tilesM, g.ntM, s, cnt * mf * mf * nf);
    // V^T = G^T P_L -> S16 and V -> T16, fp16 pairs at the scale of the bound max|G| |P_L|_1
    launch_bound_scale(cnt, g.gscale + s0, g.pln1 + s0, g.sscale + s0, g.tscale + s0, s);
    px.Dhi = reinterpret_cast<float*>(g.S16 + size_t(s0) * mn);
    px.Dlo = reinterpret_cast<float*>(g.S16 + size_t(nb) * mn + size_t(s0) * mn);
    px.ldd = g.M;
    px.Thi = reinterpret_cast<float*>(g.T16 + size_t(s0) * mn);
    px.Tlo = reinterpret_cast<float*>(g.T16 + size_t(nb) * mn + size_t(s0) * mn);
    px.ldt = g.N;
    px.oscale = g.sscale + s0;
    run_gemm(bs, op16(g.GT16, nb, s0, g.N, g.M, g.gscale), op16(g.PL16, nb, s0, g.M, g.M, g.plscale), cnt, EPI_SPLIT2,
             px, nullptr, 0, s, cnt * 2.0 * nf * mf * mf);
    // R = b R + a/m V^T V
    p.alpha = float(a / double(g.m));
    p.C = at(g.R, nn, s0);
    p.ldc = g.N;
    p.c_bstride = int64_t(nn);
    const Operand vtop = op16(g.S16, nb, s0, g.N, g.M, g.sscale);
    run_gemm(bs, vtop, vtop, cnt, EPI_SYM_EMA, p, g.tilesN, g.ntN, s, cnt * nf * nf * mf);
    std::fill(g.v_ok.begin() + s0, g.v_ok.begin() + s0 + cnt, uint8_t(1));
}

void group_stats(asg_blockset* bs, Group& g, int s0, int cnt, cudaStream_t s) {
    const asg_optimizer_config& o = bs->opt;
    const double mf = g.m, nf = g.n;  // algorithmic flops use the unpadded block
    const bool ema = o.accumulation == ASG_ACCUM_EMA;
    const size_t mn = slabMN(g), mm = slabMM(g), nn = slabNN(g);
    if (f16_mode(bs)) {
        group_stats_f16(bs, g, s0, cnt, s);
        return;
    }
    GemmParams p{};
    if (!is_kl(bs)) {
        p.alpha = ema ? float(1.0 - o.beta2) : 1.f;
        p.beta = ema ? float(o.beta2) : 1.f;
        p.C = at(g.L, mm, s0);
        p.ldc = g.M;
        p.c_bstride = int64_t(mm);
        run_gemm(bs, op(at(g.Gh, mn, s0), at(g.Gl, mn, s0), g.M, g.N), op(at(g.Gh, mn, s0), at(g.Gl, mn, s0), g.M, g.N),
                 cnt, EPI_SYM_EMA, p, g.tilesM, g.ntM, s, cnt * mf * mf * nf);
        p.C = at(g.R, nn, s0);
        p.ldc = g.N;
        p.c_bstride = int64_t(nn);
        run_gemm(bs, op(at(g.GTh, mn, s0), at(g.GTl, mn, s0), g.N, g.M), op(at(g.GTh, mn, s0), at(g.GTl, mn, s0), g.N, g.M),
                 cnt, EPI_SYM_EMA, p, g.tilesN, g.ntN, s, cnt * nf * nf * mf);
        return;
    }
    // KL-Shampoo with K = F^-1 = P^2 (P = F^-1/2 is symmetric; both come from
    // one refresh with one damping, compute_refresh in oracle/): G K_R G^T =
    // W W^T with W = G P_R, and G^T K_L G = V^T V with V = P_L G. V is also
    // the update's first product (group_update), so a step costs 8 instead of
    // 10 block-GEMM units (n^3 each at m = n), and F^-1 is never stored.
    // W = G P_R -> T
    GemmParams px{};
    px.alpha = 1.f;
    px.Dhi = at(g.Th, mn, s0);
    px.Dlo = at(g.Tl, mn, s0);
    px.ldd = g.N;
    px.d_bstride = int64_t(mn);
    run_gemm(bs, op(at(g.Gh, mn, s0), at(g.Gl, mn, s0), g.M, g.N), op(at(g.PRh, nn, s0), at(g.PRl, nn, s0), g.N, g.N),
             cnt, EPI_SPLIT, px, nullptr, 0, s, cnt * 2.0 * mf * nf * nf);
    // L = b L + a/n W W^T
    const double a = ema ? (1.0 - o.beta2) : 1.0;
    p.beta = ema ? float(o.beta2) : 1.f;
    p.alpha = float(a / double(g.n));
    p.C = at(g.L, mm, s0);
    p.ldc = g.M;
    p.c_bstride = int64_t(mm);
    run_gemm(bs, op(at(g.Th, mn, s0), at(g.Tl, mn, s0), g.M, g.N), op(at(g.Th, mn, s0), at(g.Tl, mn, s0), g.M, g.N),
             cnt, EPI_SYM_EMA, p, g.tilesM, g.ntM, s, cnt * mf * mf * nf);
    // V^T = G^T P_L -> S ([N][M]) and V -> T ([M][N], the update's operand)
    px.Dhi = at(g.Sh, mn, s0);
    px.Dlo = at(g.Sl, mn, s0);
    px.ldd = g.M;
    px.Thi = at(g.Th, mn, s0);
    px.Tlo = at(g.Tl, mn, s0);
    px.ldt = g.N;
    run_gemm(bs, op(at(g.GTh, mn, s0), at(g.GTl, mn, s0), g.N, g.M), op(at(g.PLh, mm, s0), at(g.PLl, mm, s0), g.M, g.M),
             cnt, EPI_SPLIT2, px, nullptr, 0, s, cnt * 2.0 * nf * mf * mf);
    // R = b R + a/m V^T V
    p.alpha = float(a / double(g.m));
    p.C = at(g.R, nn, s0);
    p.ldc = g.N;
    p.c_bstride = int64_t(nn);
    run_gemm(bs, op(at(g.Sh, mn, s0), at(g.Sl, mn, s0), g.N, g.M), op(at(g.Sh, mn, s0), at(g.Sl, mn, s0), g.N, g.M),
             cnt, EPI_SYM_EMA, p, g.tilesN, g.ntN, s, cnt * nf * nf * mf);
    std::fill(g.v_ok.begin() + s0, g.v_ok.begin() + s0 + cnt, uint8_t(1));
}

// accumulate_factors (precond.cpp:173-189) for every owned block: gradient
// prep (gather, clip scale, tf32 split, transpose) and the statistics GEMMs,
// batched per shape group.
void accumulate_impl(asg_blockset* bs, double clip_scale) {
    const int k = fork_groups(bs);
    for (size_t gi = 0; gi < bs->groups.size(); ++gi) {
        Group& g = bs->groups[gi];
        cudaStream_t gs = stream_for(bs, k, int(gi));
        // 4 B read per element, hi/lo of G and G^T written (16 B; 8 B in TF32 mode) per padded element
        const double bytes = double(g.nb) * (4.0 * g.m * g.n + (g.Gl ? 16.0 : 8.0) * g.M * g.N);
        hbm_launch(bs, gs, ASG_HBM_PREP, bytes, [&] {
            static const bool pred_on = !(getenv("ASG_F16_PRED") && atoi(getenv("ASG_F16_PRED")) == 0);  // A/B knob
            if (f16_mode(bs) && pred_on && g.vec_grad && g.M % 64 == 0 && g.N % 64 == 0)
                // G, G^T as fp16 pairs (8 B/elt written) at the scale predicted from the last
                // step's max, the max fused in; mispredicted blocks rewritten
                launch_prep_grad_f16_pred(g.d_refs, g.nb, g.M, g.N, float(clip_scale), g.amaxp, g.amax2, g.gfix, g.G16,
                                          g.G16 + size_t(g.nb) * slabMN(g), g.GT16,
                                          g.GT16 + size_t(g.nb) * slabMN(g), g.gscale, gs);
            else if (f16_mode(bs))  // (+ a 4 B/elt max pass)
                launch_prep_grad_f16(g.d_refs, g.nb, g.M, g.N, float(clip_scale), g.amax2, g.G16,
                                     g.G16 + size_t(g.nb) * slabMN(g), g.GT16, g.GT16 + size_t(g.nb) * slabMN(g),
                                     g.gscale, gs, g.vec_grad);
            else
                launch_prep_grad(g.d_refs, g.nb, g.M, g.N, nullptr, float(clip_scale), g.Gh, g.Gl, g.GTh, g.GTl, gs,
                                 g.vec_grad);
        });
        group_stats(bs, g, 0, g.nb, gs);
    }
    join_groups(bs, k);
}

// Preconditioned update for slots [s0, s0+cnt). `final_epi` is EPI_APPLY (step)
// or EPI_STORE into `store_out` ([cnt][M][N], parity entry points).
void group_update(asg_blockset* bs, Group& g, int s0, int cnt, int final_epi, float lr_eff, const ApplyEntry* apply,
                  float* store_out, cudaStream_t s) {
    const asg_optimizer_config& o = bs->opt;
    const double mf = g.m, nf = g.n;
    const size_t mn = slabMN(g), mm = slabMM(g), nn = slabNN(g);
    GemmParams pf{};
    pf.alpha = 1.f;
    pf.beta = 0.f;
    pf.apply = apply;
    pf.lr_eff = lr_eff;
    pf.wd = float(o.weight_decay);
    pf.flag = bs->d_upd_flag;
    pf.C = store_out;
    pf.ldc = g.N;
    pf.c_bstride = int64_t(mn);
    GemmParams ps{};
    ps.alpha = 1.f;
    ps.ldd = g.N;
    ps.d_bstride = int64_t(mn);
    if (!is_soap(bs)) {
        // Y = P_L G -> T ; U = Y P_R. KL-Shampoo: T already holds V = P_L G
        // from the statistics (group_stats) for the slots whose roots and
        // gradient are unchanged since; only the others are recomputed.
        int r0 = s0, r1 = s0 + cnt;
        if (is_kl(bs)) {
            while (r0 < r1 && g.v_ok[size_t(r0)]) ++r0;
            while (r1 > r0 && g.v_ok[size_t(r1 - 1)]) --r1;
        }
        if (f16_mode(bs)) {
            const int nb = g.nb;
            if (r1 > r0) {
                launch_bound_scale(r1 - r0, g.gscale + r0, g.pln1 + r0, g.tscale + r0, nullptr, s);
                ps.Dhi = reinterpret_cast<float*>(g.T16 + size_t(r0) * mn);
                ps.Dlo = reinterpret_cast<float*>(g.T16 + size_t(nb) * mn + size_t(r0) * mn);
                ps.oscale = g.tscale + r0;
                run_gemm(bs, op16(g.PL16, nb, r0, g.M, g.M, g.plscale), op16(g.GT16, nb, r0, g.N, g.M, g.gscale),
                         r1 - r0, EPI_SPLIT, ps, nullptr, 0, s, (r1 - r0) * 2.0 * mf * mf * nf);
                if (is_kl(bs)) std::fill(g.v_ok.begin() + r0, g.v_ok.begin() + r1, uint8_t(1));
            }
            run_gemm(bs, op16(g.T16, nb, s0, g.M, g.N, g.tscale), op16(g.PR16, nb, s0, g.N, g.N, g.prscale), cnt,
                     final_epi, pf, nullptr, 0, s, cnt * 2.0 * mf * nf * nf);
            return;
        }
        if (r1 > r0) {
            ps.Dhi = at(g.Th, mn, r0);
            ps.Dlo = at(g.Tl, mn, r0);
            run_gemm(bs, op(at(g.PLh, mm, r0), at(g.PLl, mm, r0), g.M, g.M),
                     op(at(g.GTh, mn, r0), at(g.GTl, mn, r0), g.N, g.M), r1 - r0, EPI_SPLIT, ps, nullptr, 0, s,
                     (r1 - r0) * 2.0 * mf * mf * nf);
            if (is_kl(bs)) std::fill(g.v_ok.begin() + r0, g.v_ok.begin() + r1, uint8_t(1));
        }
        run_gemm(bs, op(at(g.Th, mn, s0), at(g.Tl, mn, s0), g.M, g.N), op(at(g.PRh, nn, s0), at(g.PRl, nn, s0), g.N, g.N),
                 cnt, final_epi, pf, nullptr, 0, s, cnt * 2.0 * mf * nf * nf);
        return;
    }
    // SOAP (soap_scaled_step precond.cpp:208-223)
    const Unit& u0 = bs->units[size_t(g.units[size_t(s0)])];
    const double t = double(u0.moment_steps);  // already incremented by the caller
    GemmParams pa{};
    pa.alpha = 1.f;
    pa.Dhi = at(g.Sh, mn, s0);
    pa.Dlo = at(g.Sl, mn, s0);
    pa.ldd = g.N;
    pa.d_bstride = int64_t(mn);
    pa.mom_m = at(g.mom_m, mn, s0);
    pa.mom_v = at(g.mom_v, mn, s0);
    pa.ldm = g.N;
    pa.m_bstride = int64_t(mn);
    pa.b1 = float(o.beta1);
    pa.b2 = float(o.beta2);
    pa.inv_bc1 = float(1.0 / (1.0 - std::pow(o.beta1, t)));
    pa.inv_bc2 = float(1.0 / (1.0 - std::pow(o.beta2, t)));
    pa.adam_eps = float(o.eps);
    // T = Q_L^T G
    ps.Dhi = at(g.Th, mn, s0);
    ps.Dlo = at(g.Tl, mn, s0);
    run_gemm(bs, op(at(g.QLTh, mm, s0), at(g.QLTl, mm, s0), g.M, g.M), op(at(g.GTh, mn, s0), at(g.GTl, mn, s0), g.N, g.M),
             cnt, EPI_SPLIT, ps, nullptr, 0, s, cnt * 2.0 * mf * mf * nf);
    // Adam(T Q_R) -> S
    run_gemm(bs, op(at(g.Th, mn, s0), at(g.Tl, mn, s0), g.M, g.N), op(at(g.QRTh, nn, s0), at(g.QRTl, nn, s0), g.N, g.N),
             cnt, EPI_ADAM, pa, nullptr, 0, s, cnt * 2.0 * mf * nf * nf);
    // W^T = (S Q_R^T)^T -> T as [N][M]
    GemmParams pt{};
    pt.alpha = 1.f;
    pt.Dhi = at(g.Th, mn, s0);
    pt.Dlo = at(g.Tl, mn, s0);
    pt.ldd = g.M;
    pt.d_bstride = int64_t(mn);
    run_gemm(bs, op(at(g.Sh, mn, s0), at(g.Sl, mn, s0), g.M, g.N), op(at(g.QRh, nn, s0), at(g.QRl, nn, s0), g.N, g.N),
             cnt, EPI_SPLIT_T, pt, nullptr, 0, s, cnt * 2.0 * mf * nf * nf);
    // U = Q_L W
    run_gemm(bs, op(at(g.QLh, mm, s0), at(g.QLl, mm, s0), g.M, g.M), op(at(g.Th, mn, s0), at(g.Tl, mn, s0), g.N, g.M),
             cnt, final_epi, pf, nullptr, 0, s, cnt * 2.0 * mf * mf * nf);
}

// ---------------------------------------------------------------------------
// refresh (side stream) and install (main stream)
// ---------------------------------------------------------------------------
// One side of one chunk: factor slab slots [s0, s0+cnt) of dim d (padded D).
void refresh_side(asg_blockset* bs, Group& g, int s0, int cnt, bool left, cudaStream_t s) {
    const int d = left ? g.m : g.n, D = left ? g.M : g.N;
    const size_t DD = size_t(D) * D, dd = size_t(d) * d;
    const float* snap = at(left ? g.snapL : g.snapR, DD, s0);
    launch_snapshot(snap, cnt, D, d, bs->ws_snap, s);
    // Warm start from the block's previous eigenbasis once every block of the
    // chunk has one (the result does not depend on the start; only the sweep
    // count does).
    bool warm = true;
    for (int k = 0; k < cnt; ++k) warm &= bs->units[size_t(g.units[size_t(s0 + k)])].warm_start;
    const double* prev = nullptr;
    if (warm) prev = is_soap(bs) ? at(left ? g.QL64 : g.QR64, dd, s0) : at(left ? g.EL64 : g.ER64, dd, s0);
    launch_eigh(bs->ws_snap, bs->ws_vals, bs->ws_vecs, bs->ws_work, cnt, d, g.d_status + s0, s, prev);
    if (!is_soap(bs))
        CK(cudaMemcpyAsync(at(left ? g.EL64 : g.ER64, dd, s0), bs->ws_vecs, size_t(cnt) * dd * 8,
                           cudaMemcpyDeviceToDevice, s));
    if (is_soap(bs)) {
        CK(cudaMemcpyAsync(at(left ? g.sQL64 : g.sQR64, dd, s0), bs->ws_vecs, size_t(cnt) * dd * 8,
                           cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(at(left ? g.svalsL : g.svalsR, size_t(d), s0), bs->ws_vals, size_t(cnt) * d * 8,
                           cudaMemcpyDeviceToDevice, s));
        return;
    }
    launch_relative_damping(bs->ws_snap, cnt, d, bs->opt.damping, bs->ws_eps, s);
    struct Out {
        double power;
        float *hi, *lo;
    };
    // Shampoo F^-1/4, KL-Shampoo F^-1/2 (its F^-1 = (F^-1/2)^2 is not stored)
    const Out outs[1] = {{is_kl(bs) ? -0.5 : -0.25, at(left ? g.sPLh : g.sPRh, DD, s0),
                          at(left ? g.sPLl : g.sPRl, DD, s0)}};
    for (const Out& o : outs) {
        launch_scale_columns(bs->ws_vecs, bs->ws_vals, bs->ws_eps, o.power, cnt, d, bs->ws_W, g.d_status + s0, s);
        // V diag(w) V^T  (densela.hpp:280), symmetrized on conversion
        launch_dgemm(false, true, d, d, d, 1.0, bs->ws_W, d, int64_t(dd), bs->ws_vecs, d, int64_t(dd), 0.0, bs->ws_out,
                     d, int64_t(dd), cnt, s);
        launch_f64_to_split(bs->ws_out, cnt, d, D, true, o.hi, o.lo, nullptr, nullptr, s);
    }
}


// Newton-Schulz re-orthonormalization of Q J is needed after a cold solve (J
// carries the tensor-core Jacobi's accumulated rounding) and periodically
// after warm ones (each product adds ~1e-7 of drift): every kNsPeriod-th
// refresh of a block.
constexpr uint64_t kNsPeriod = 8;
bool needs_ns(const asg_blockset* bs, const Group& g, int s0, int cnt, bool at_install) {
    for (int k = 0; k < cnt; ++k) {
        const Unit& u = bs->units[size_t(g.units[size_t(s0 + k)])];
        // refresh: version before this job's install; install: version already bumped
        const uint64_t v = at_install ? (u.version ? u.version - 1 : 0) : u.version;
        if (!u.warm_start || v % kNsPeriod == 0) return true;
    }
    return false;
}

// One Newton-Schulz polar step on a split basis slab (cnt blocks of D x D):
// out = V (3 I - V^T V) / 2. VT: scratch for V^T (split), Sx: fp32 scratch
// reused in place for X's hi part, Xl: X's lo part (null in TF32 mode).
void orthonormalize(asg_blockset* bs, const float* Vh, const float* Vl, float* outh, float* outl, float* VTh,
                    float* VTl, float* Sx, float* Xl, int cnt, int d, int D, const int2* sym_tiles, int nsym,
                    cudaStream_t s) {
    const size_t DD = size_t(D) * D;
    const double flops = 2.0 * cnt * double(d) * d * d;
    launch_transpose_split(Vh, Vl, cnt, D, D, VTh, VTl, false, s);
    GemmParams p1{};
    p1.alpha = 1.f;
    p1.beta = 0.f;
    p1.C = Sx;
    p1.ldc = D;
    p1.c_bstride = int64_t(DD);
    // V^T V is symmetric: lower-triangle tiles + mirror
    run_gemm(bs, op(VTh, VTl, D, D), op(VTh, VTl, D, D), cnt, EPI_SYM_EMA, p1, sym_tiles, nsym, s, flops / 2);
    launch_ns_x(Sx, cnt, d, D, Sx, Xl, s);
    GemmParams p2{};
    p2.alpha = 1.f;
    p2.Dhi = outh;
    p2.Dlo = outl;
    p2.ldd = D;
    p2.d_bstride = int64_t(DD);
    run_gemm(bs, op(Vh, Vl, D, D), op(Sx, Xl, D, D), cnt, EPI_SPLIT, p2, nullptr, 0, s, flops);
}

// F32 refresh of one side of one chunk (asg_refresh_mode F32). With Q the
// block's previous eigenbasis (identity before the first refresh):
//   B = Q^T A Q (two 3xTF32 GEMMs), J = eig(B) (fp64 block Jacobi, relative
//   threshold), then Shampoo/KL: V = Q J becomes the new basis and the roots
//   V f(lambda) V^T are GEMMs; SOAP: J^T is kept as the shadow rotation, the
//   install forms Q J and re-projects the moments (install_soap_f32).
// ASG_REFRESH_TIMING=1: per refresh chunk, host-synchronous phase timings on
// the side stream (diagnostics only; breaks the overlap with the main stream).
struct PhaseTimer {
    bool on;
    cudaStream_t s;
    std::vector<std::pair<const char*, cudaEvent_t>> marks;
    explicit PhaseTimer(cudaStream_t st) : on(getenv("ASG_REFRESH_TIMING") != nullptr), s(st) {}
    void mark(const char* name) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        marks.emplace_back(name, e);
    }
    void report(int d, int cnt) {
        if (!on || marks.size() < 2) return;
        cudaEventSynchronize(marks.back().second);
        std::fprintf(stderr, "refresh d=%d cnt=%d:", d, cnt);
        for (size_t i = 1; i < marks.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
            std::fprintf(stderr, " %s %.3f", marks[i].first, ms);
        }
        std::fprintf(stderr, " ms\n");
        for (auto& m : marks) cudaEventDestroy(m.second);
    }
};

// F32 refresh of one chunk of a group: both factor sides in one batched
// eigensolve when they have the same dimension (square blocks), else one side.
void refresh_sides_f32(asg_blockset* bs, Group& g, int s0, int cnt, int nsides, bool first_left, cudaStream_t s) {
    PhaseTimer pt(s);
    pt.mark("start");
    const int d = first_left ? g.m : g.n, D = first_left ? g.M : g.N;
    const size_t DD = size_t(D) * D, cntDD = size_t(cnt) * DD;
    const double dd3 = double(cnt) * d * double(d) * d;
    const int nb = nsides * cnt;  // matrices in the eigensolve
    float** t = bs->tw;
    const bool sp = split_mode(bs);
    auto off = [&](float* base, int j) { return base ? base + size_t(j) * cntDD : nullptr; };
    struct Side {
        bool left;
        float *Qh, *Ql, *QTh, *QTl;
        const int2* tiles;
        int ntiles;
    };
    std::vector<Side> sides;
    for (int j = 0; j < nsides; ++j) {
        const bool left = nsides == 2 ? j == 0 : first_left;
        Side sd{};
        sd.left = left;
        if (is_soap(bs)) {
            sd.Qh = at(left ? g.QLh : g.QRh, DD, s0);
            sd.Ql = at(left ? g.QLl : g.QRl, DD, s0);
            sd.QTh = at(left ? g.QLTh : g.QRTh, DD, s0);
            sd.QTl = at(left ? g.QLTl : g.QRTl, DD, s0);
        } else {
            sd.Qh = at(left ? g.BLh : g.BRh, DD, s0);
            sd.Ql = at(left ? g.BLl : g.BRl, DD, s0);
            sd.QTh = at(left ? g.BLTh : g.BRTh, DD, s0);
            sd.QTl = at(left ? g.BLTl : g.BRTl, DD, s0);
        }
        sd.tiles = left ? g.tilesM : g.tilesN;
        sd.ntiles = left ? g.ntM : g.ntN;
        sides.push_back(sd);
    }
    // per side j: A_j split -> t0/t1[j], W_j^T = (A_j Q_j)^T -> t2/t3[j], B_j = Q_j^T W_j -> t4[j]
    for (int j = 0; j < nsides; ++j) {
        const Side& sd = sides[size_t(j)];
        const float* snap = at(sd.left ? g.snapL : g.snapR, DD, s0);
        if (sp) launch_split_slab(snap, off(t[0], j), off(t[1], j), int64_t(cntDD), s);
        else CK(cudaMemcpyAsync(off(t[0], j), snap, cntDD * 4, cudaMemcpyDeviceToDevice, s));
        GemmParams p1{};
        p1.alpha = 1.f;
        p1.Dhi = off(t[2], j);
        p1.Dlo = sp ? off(t[3], j) : nullptr;
        p1.ldd = D;
        p1.d_bstride = int64_t(DD);
        run_gemm(bs, op(off(t[0], j), sp ? off(t[1], j) : nullptr, D, D), op(sd.QTh, sd.QTl, D, D), cnt, EPI_SPLIT_T,
                 p1, nullptr, 0, s, 2.0 * dd3);
        GemmParams p2{};
        p2.alpha = 1.f;
        p2.beta = 0.f;
        p2.C = off(t[4], j);
        p2.ldc = D;
        p2.c_bstride = int64_t(DD);
        // B = Q^T A Q is symmetric: lower-triangle tiles + mirror (exactly symmetric output)
        run_gemm(bs, op(sd.QTh, sd.QTl, D, D), op(off(t[2], j), sp ? off(t[3], j) : nullptr, D, D), cnt, EPI_SYM_EMA,
                 p2, sd.tiles, sd.ntiles, s, dd3);
    }
    pt.mark("transform");
    // relative damping eps = damping * tr(B) / d (tr B = tr A: orthogonal similarity)
    launch_relative_damping_f32(t[4], nb, D, d, bs->opt.damping, bs->ws_eps, s);
    int* st = nsides == 2 ? bs->pair_status : g.d_status + s0;
    if (nsides == 2) CK(cudaMemsetAsync(st, 0, size_t(nb) * sizeof(int), s));
    float* t1 = work_split(bs) ? t[1] : nullptr;
    float* t3 = work_split(bs) ? t[3] : nullptr;
    if (d > kSmallEighN && !bs->fp64_jacobi) {
        // tensor-core block Jacobi over all sides: J -> (t0, t1), J^T -> (t2, t3)
        // (Q J is re-orthonormalized below / at the SOAP install, so J itself is not)
        launch_tc_eigh(t[4], D, bs->ws_vals, t[0], t1, t[2], t3, bs->tc_ws, nb, d, st, bs->num_sms, s,
                       f32_refresh_tol(), false, g.d_identL ? bs->pair_ident : nullptr);
    } else {
        launch_snapshot_sym(t[4], nb, D, d, bs->ws_snap, s);
        EighOpts eo;
        eo.relative = 1;
        eo.tol = f32_refresh_tol();
        launch_eigh(bs->ws_snap, bs->ws_vals, bs->ws_vecs, bs->ws_work, nb, d, st, s, nullptr, eo);
        launch_f64_to_split(bs->ws_vecs, nb, d, D, false, t[0], t1, t[2], t3, s);
        if (g.d_identL) CK(cudaMemsetAsync(bs->pair_ident, 0, size_t(nb) * sizeof(int), s));  // unknown: full install
    }
    if (g.d_identL)
        for (int j = 0; j < nsides; ++j)
            CK(cudaMemcpyAsync((sides[size_t(j)].left ? g.d_identL : g.d_identR) + s0, bs->pair_ident + size_t(j) * cnt,
                               size_t(cnt) * sizeof(int), cudaMemcpyDeviceToDevice, s));
    if (nsides == 2) launch_merge_status(st, cnt, g.d_status + s0, s);
    pt.mark("eigh");
    for (int j = 0; j < nsides; ++j) {
        const Side& sd = sides[size_t(j)];
        const bool left = sd.left;
        const double* vals = bs->ws_vals + size_t(j) * cnt * d;
        if (is_soap(bs)) {
            if (sp || !t3) {
                CK(cudaMemcpyAsync(at(left ? g.sJLTh : g.sJRTh, DD, s0), off(t[2], j), cntDD * 4,
                                   cudaMemcpyDeviceToDevice, s));
                if (sp)
                    CK(cudaMemcpyAsync(at(left ? g.sJLTl : g.sJRTl, DD, s0), off(t[3], j), cntDD * 4,
                                       cudaMemcpyDeviceToDevice, s));
            } else {  // 3XTF32_SMEM: the shadow rotation is stored as plain fp32 (hi + lo)
                launch_merge_pair(off(t[2], j), off(t[3], j), at(left ? g.sJLTh : g.sJRTh, DD, s0), int64_t(cntDD), s);
            }
            CK(cudaMemcpyAsync(at(left ? g.svalsL : g.svalsR, size_t(d), s0), vals, size_t(cnt) * d * 8,
                               cudaMemcpyDeviceToDevice, s));
            continue;
        }
        // V = Q J -> (t4, t5)[j] (B is no longer needed); it becomes the block's basis
        float* V = off(t[4], j);
        float* Vl = sp ? off(t[5], j) : nullptr;
        GemmParams p3{};
        p3.alpha = 1.f;
        p3.Dhi = V;
        p3.Dlo = Vl;
        p3.ldd = D;
        p3.d_bstride = int64_t(DD);
        run_gemm(bs, op(sd.Qh, sd.Ql, D, D), op(off(t[2], j), t3 ? off(t[3], j) : nullptr, D, D), cnt, EPI_SPLIT, p3,
                 nullptr, 0, s, 2.0 * dd3);
        // re-orthonormalize (the products drift at the fp32 level), straight into the basis
        if (needs_ns(bs, g, s0, cnt, false)) {
            orthonormalize(bs, V, Vl, sd.Qh, sp ? sd.Ql : nullptr, off(t[2], j), sp ? off(t[3], j) : nullptr,
                           off(t[6], j), sp ? off(t[7], j) : nullptr, cnt, d, D, sd.tiles, sd.ntiles, s);
            CK(cudaMemcpyAsync(V, sd.Qh, cntDD * 4, cudaMemcpyDeviceToDevice, s));
            if (sp) CK(cudaMemcpyAsync(Vl, sd.Ql, cntDD * 4, cudaMemcpyDeviceToDevice, s));
        } else {
            CK(cudaMemcpyAsync(sd.Qh, V, cntDD * 4, cudaMemcpyDeviceToDevice, s));
            if (sp) CK(cudaMemcpyAsync(sd.Ql, Vl, cntDD * 4, cudaMemcpyDeviceToDevice, s));
        }
        launch_transpose_split(V, Vl, cnt, D, D, sd.QTh, sp ? sd.QTl : nullptr, false, s);
        // roots V diag((lambda + eps)^p) V^T  (inv_root densela.hpp:267-282, damping precond.cpp:121-125)
        struct Out {
            double power;
            float *hi, *lo;
        };
        const Out outs[1] = {{is_kl(bs) ? -0.5 : -0.25, at(left ? g.sPLh : g.sPRh, DD, s0),
                              at(left ? g.sPLl : g.sPRl, DD, s0)}};
        for (const Out& o : outs) {
            launch_scale_columns_split(V, Vl, vals, bs->ws_eps + size_t(j) * cnt, o.power, cnt, d, D, off(t[6], j),
                                       sp ? off(t[7], j) : nullptr, g.d_status + s0, s);
            GemmParams pr{};
            pr.alpha = 1.f;
            pr.Dhi = o.hi;
            pr.Dlo = o.lo;
            pr.ldd = D;
            pr.d_bstride = int64_t(DD);
            run_gemm(bs, op(off(t[6], j), sp ? off(t[7], j) : nullptr, D, D), op(V, Vl, D, D), cnt, EPI_SPLIT, pr,
                     nullptr, 0, s, 2.0 * dd3);
        }
    }
    pt.mark("basis+roots");
    pt.report(d, nb);
}

// NEWTON refresh of one chunk (Shampoo / KL-Shampoo): per side, the damped
// snapshot's inverse root by coupled Newton-Schulz straight into the shadow
// roots (compute_refresh precond.cpp:136-140: inv_root(F, 4, damping tr/n));
// KL-Shampoo's F^-1 is (F^-1/2)^2 and is never formed (group_stats).
void refresh_newton(asg_blockset* bs, Group& g, int s0, int cnt, cudaStream_t s) {
    PhaseTimer pt(s);
    pt.mark("start");
    // square blocks whose whole group is this chunk: both sides in one batch
    // (the jointly allocated L/R slabs are contiguous), which halves the
    // iteration's latency when the group is small (C1: one 1024^2 block)
    const bool both = g.m == g.n && s0 == 0 && cnt == g.nb && g.nb <= bs->ws_chunk;
    for (int side = 0; side < (both ? 1 : 2); ++side) {
        const bool left = side == 0;
        const int d = left ? g.m : g.n, D = left ? g.M : g.N;
        const int nmat = both ? 2 * cnt : cnt;
        const size_t DD = size_t(D) * D;
        const float* snap = at(left ? g.snapL : g.snapR, DD, s0);
        launch_relative_damping_f32(snap, nmat, D, d, bs->opt.damping, bs->ws_eps, s);
        float* ph = at(left ? g.sPLh : g.sPRh, DD, s0);
        float* pl = at(left ? g.sPLl : g.sPRl, DD, s0);
        const int2* tiles = left ? g.tilesM : g.tilesN;
        const int ntiles = left ? g.ntM : g.ntN;
        int* st = both ? bs->pair_status : g.d_status + s0;
        if (both) CK(cudaMemsetAsync(st, 0, size_t(nmat) * sizeof(int), s));
        launch_ns_inv_root(snap, nmat, d, D, bs->ws_eps, is_kl(bs) ? 2 : 4, ph, pl, bs->ns_ws, st, tiles, ntiles,
                           bs->precision, bs->num_sms, s);
        if (both) launch_merge_status(st, cnt, g.d_status + s0, s);
    }
    pt.mark("newton roots");
    pt.report(g.m, cnt);
}

// Launches the refresh for every unit marked dispatched-but-not-launched.
void launch_refreshes(asg_blockset* bs) {
    std::vector<std::vector<int>> per_group(bs->groups.size());
    for (size_t i = 0; i < bs->units.size(); ++i) {
        Unit& u = bs->units[i];
        if (u.needs_launch && u.group >= 0) per_group[size_t(u.group)].push_back(int(i));
    }
    bool any = false;
    for (auto& v : per_group) any |= !v.empty();
    if (!any) return;
    // snapshot on the main stream (after this step's accumulation), then the
    // side stream works from the snapshot (snapshot isolation, asyncsched.cpp:129-136)
    for (size_t gi = 0; gi < bs->groups.size(); ++gi) {
        Group& g = bs->groups[gi];
        // one copy per contiguous slot run (a dispatch step snapshots hundreds of blocks)
        std::vector<int> sl;
        for (int ui : per_group[gi])
            if (!bs->units[size_t(ui)].snap_preloaded) sl.push_back(bs->units[size_t(ui)].slot);
        std::sort(sl.begin(), sl.end());
        for (size_t a = 0; a < sl.size();) {
            size_t b = a + 1;
            while (b < sl.size() && sl[b] == sl[b - 1] + 1) ++b;
            const size_t cnt = b - a;
            CK(cudaMemcpyAsync(at(g.snapL, slabMM(g), sl[a]), at(g.L, slabMM(g), sl[a]), cnt * slabMM(g) * 4,
                               cudaMemcpyDeviceToDevice, bs->main));
            CK(cudaMemcpyAsync(at(g.snapR, slabNN(g), sl[a]), at(g.R, slabNN(g), sl[a]), cnt * slabNN(g) * 4,
                               cudaMemcpyDeviceToDevice, bs->main));
            a = b;
        }
        for (int ui : per_group[gi]) bs->units[size_t(ui)].snap_preloaded = false;
    }
    CK(cudaEventRecord(bs->ev_snap, bs->main));
    CK(cudaStreamWaitEvent(bs->side, bs->ev_snap, 0));
    if (bs->nside == 2) CK(cudaStreamWaitEvent(bs->side2, bs->ev_snap, 0));
    int chunk_no = 0;  // chunks alternate between the side streams (own workspace sets)
    for (size_t gi = 0; gi < bs->groups.size(); ++gi) {
        Group& g = bs->groups[gi];
        std::vector<int> slots;
        for (int ui : per_group[gi]) slots.push_back(bs->units[size_t(ui)].slot);
        std::sort(slots.begin(), slots.end());
        size_t i = 0;
        while (i < slots.size()) {
            // maximal contiguous run, split into workspace-sized chunks
            size_t j = i + 1;
            while (j < slots.size() && slots[j] == slots[j - 1] + 1 && int(j - i) < bs->ws_chunk) ++j;
            const int s0 = slots[i], cnt = int(j - i);
            const int lane = bs->nside == 2 ? (chunk_no++ & 1) : 0;
            cudaStream_t sst = lane ? bs->side2 : bs->side;
            load_side_ws(bs, bs->side_ws[lane]);
            CK(cudaMemsetAsync(g.d_status + s0, 0, size_t(cnt) * sizeof(int), sst));
            if (newton_roots(bs)) {
                refresh_newton(bs, g, s0, cnt, sst);
            } else if (f32_refresh(bs)) {
                if (g.m == g.n && g.m > kSmallEighN && !bs->fp64_jacobi) {
                    refresh_sides_f32(bs, g, s0, cnt, 2, true, sst);
                } else {
                    refresh_sides_f32(bs, g, s0, cnt, 1, true, sst);
                    refresh_sides_f32(bs, g, s0, cnt, 1, false, sst);
                }
            } else {
                refresh_side(bs, g, s0, cnt, true, sst);
                refresh_side(bs, g, s0, cnt, false, sst);
            }
            CK(cudaMemcpyAsync(g.h_status + s0, g.d_status + s0, size_t(cnt) * sizeof(int), cudaMemcpyDeviceToHost,
                               sst));
            if (g.d_identL) {
                CK(cudaMemcpyAsync(g.h_identL + s0, g.d_identL + s0, size_t(cnt) * sizeof(int), cudaMemcpyDeviceToHost,
                                   sst));
                CK(cudaMemcpyAsync(g.h_identR + s0, g.d_identR + s0, size_t(cnt) * sizeof(int), cudaMemcpyDeviceToHost,
                                   sst));
            }
            for (int k = 0; k < cnt; ++k) {
                Unit& u = bs->units[size_t(g.units[size_t(s0 + k)])];
                CK(cudaEventRecord(u.done, sst));
                u.launched = true;
                u.needs_launch = false;
            }
            i = j;
        }
    }
    load_side_ws(bs, bs->side_ws[0]);
    CK(cudaGetLastError());
}

int status_to_code(int st) { return st; }

// Orders the install after a unit's refresh. A refresh that has completed is
// installed at once (its status checked now). Otherwise, in EVENT mode, the
// main stream waits on the refresh event (no host blocking, SURVEY 8(b)
// threading row) and the status and device-side wait are resolved at the
// next host sync (resolve_deferred); in SIM_CLOCK mode (deterministic parity
// runs) and for the synchronous per-block entry points the host waits and a
// failed refresh throws here, as future.get() does (asyncsched.cpp:146).
void install_wait(asg_blockset* bs, Unit& u, bool host_wait) {
    if (u.needs_launch) launch_refreshes(bs);
    Group& g = bs->groups[size_t(u.group)];
    const cudaError_t q = cudaEventQuery(u.done);
    if (q != cudaSuccess && q != cudaErrorNotReady) CK(q);
    if (q == cudaErrorNotReady && !host_wait) {
        asg_blockset::DeferredInstall d{int(&u - bs->units.data()), nullptr, nullptr};
        CK(cudaEventCreate(&d.ev_a));
        CK(cudaEventCreate(&d.ev_b));
        CK(cudaEventRecord(d.ev_a, bs->main));
        CK(cudaStreamWaitEvent(bs->main, u.done, 0));
        CK(cudaEventRecord(d.ev_b, bs->main));
        bs->deferred_status.push_back(d);
        return;
    }
    if (q == cudaErrorNotReady) CK(cudaEventSynchronize(u.done));
    const int st = g.h_status[u.slot];
    if (st != ASG_OK) {
        const char* what = st == ASG_ERR_NOT_PSD       ? "refresh: damped eigenvalue <= 0"
                           : st == ASG_ERR_NON_FINITE   ? "refresh: non-finite factor"
                           : st == ASG_ERR_NO_CONVERGENCE ? "refresh: eigensolver sweep budget exhausted"
                                                          : "refresh failed";
        throw Fail{status_to_code(st), what};
    }
}

// SOAP install of the F32 refresh for slots [s0, s0+cnt) of a group
// (install_refresh precond.cpp:145-157 with rot = Q_new^T Q_old = J^T):
//   Q <- Q J ;  M <- J_L^T M J_R ;  V <- (J_L o J_L)^T V (J_R o J_R) ;  values.
void install_soap_f32(asg_blockset* bs, Group& g, int s0, int cnt) {
    cudaStream_t s = bs->main;
    const bool ns = needs_ns(bs, g, s0, cnt, true);
    const bool sp = split_mode(bs);
    float** w = bs->iw32;
    const size_t MN = slabMN(g);
    for (int side = 0; side < 2; ++side) {
        const bool left = side == 0;
        const int d = left ? g.m : g.n, D = left ? g.M : g.N;
        const size_t DD = size_t(D) * D;
        float* Qh = at(left ? g.QLh : g.QRh, DD, s0);
        float* Ql = at(left ? g.QLl : g.QRl, DD, s0);
        GemmParams p{};
        p.alpha = 1.f;
        p.Dhi = w[0];
        p.Dlo = sp ? w[1] : nullptr;
        p.ldd = D;
        p.d_bstride = int64_t(DD);
        run_gemm(bs, op(Qh, Ql, D, D), op(at(left ? g.sJLTh : g.sJRTh, DD, s0), at(left ? g.sJLTl : g.sJRTl, DD, s0), D, D),
                 cnt, EPI_SPLIT, p, nullptr, 0, s, 2.0 * cnt * double(d) * d * d);
        // Q <- orthonormalized (Q_old J), then Q^T
        if (ns) {
            orthonormalize(bs, w[0], sp ? w[1] : nullptr, Qh, sp ? Ql : nullptr, w[2], sp ? w[3] : nullptr, w[4],
                           sp ? w[5] : nullptr, cnt, d, D, left ? g.tilesM : g.tilesN, left ? g.ntM : g.ntN, s);
        } else {
            CK(cudaMemcpyAsync(Qh, w[0], size_t(cnt) * DD * 4, cudaMemcpyDeviceToDevice, s));
            if (sp) CK(cudaMemcpyAsync(Ql, w[1], size_t(cnt) * DD * 4, cudaMemcpyDeviceToDevice, s));
        }
        launch_transpose_split(Qh, sp ? Ql : nullptr, cnt, D, D, at(left ? g.QLTh : g.QRTh, DD, s0),
                               at(left ? g.QLTl : g.QRTl, DD, s0), false, s);
        CK(cudaMemcpyAsync(at(left ? g.valsL : g.valsR, size_t(d), s0), at(left ? g.svalsL : g.svalsR, size_t(d), s0),
                           size_t(cnt) * d * 8, cudaMemcpyDeviceToDevice, s));
    }
    const size_t mm = slabMM(g), nn = slabNN(g);
    const double flops = 2.0 * cnt * double(g.m) * g.n * (g.m + g.n);
    for (int which = 0; which < 2; ++which) {
        float* mom = at(which == 0 ? g.mom_m : g.mom_v, MN, s0);
        const float *lh = at(g.sJLTh, mm, s0), *ll = at(g.sJLTl, mm, s0);
        const float *rh = at(g.sJRTh, nn, s0), *rl = at(g.sJRTl, nn, s0);
        if (which == 1) {  // elementwise squares of the rotations
            launch_square_split(lh, ll, w[0], sp ? w[1] : nullptr, int64_t(size_t(cnt) * mm), s);
            launch_square_split(rh, rl, w[2], sp ? w[3] : nullptr, int64_t(size_t(cnt) * nn), s);
            lh = w[0];
            ll = sp ? w[1] : nullptr;
            rh = w[2];
            rl = sp ? w[3] : nullptr;
        }
        // M^T as the B operand (S slabs are free outside the update)
        launch_transpose_split(mom, nullptr, cnt, g.M, g.N, at(g.Sh, MN, s0), at(g.Sl, MN, s0), false, s);
        GemmParams pt{};
        pt.alpha = 1.f;
        pt.Dhi = at(g.Th, MN, s0);
        pt.Dlo = at(g.Tl, MN, s0);
        pt.ldd = g.N;
        pt.d_bstride = int64_t(MN);
        run_gemm(bs, op(lh, ll, g.M, g.M), op(at(g.Sh, MN, s0), at(g.Sl, MN, s0), g.N, g.M), cnt, EPI_SPLIT, pt, nullptr,
                 0, s, 2.0 * cnt * double(g.m) * g.m * g.n);
        GemmParams po{};
        po.alpha = 1.f;
        po.beta = 0.f;
        po.C = mom;
        po.ldc = g.N;
        po.c_bstride = int64_t(MN);
        run_gemm(bs, op(at(g.Th, MN, s0), at(g.Tl, MN, s0), g.M, g.N), op(rh, rl, g.N, g.N), cnt, EPI_STORE, po, nullptr,
                 0, s, 2.0 * cnt * double(g.m) * g.n * g.n);
    }
    (void)flops;
}

// Shampoo / KL-Shampoo install for slots [s0, s0+cnt) of a group
// (install_refresh precond.cpp:158-161): shadow roots -> active, one copy per
// array over the whole slot run.
void install_roots(asg_blockset* bs, Group& g, int s0, int cnt) {
    cudaStream_t s = bs->main;
    const size_t mm = slabMM(g), nn = slabNN(g);
    auto cp = [&](float* dst, const float* src, size_t n) {
        if (dst && src) CK(cudaMemcpyAsync(dst, src, n * size_t(cnt) * 4, cudaMemcpyDeviceToDevice, s));
    };
    cp(at(g.PLh, mm, s0), at(g.sPLh, mm, s0), mm);
    cp(at(g.PLl, mm, s0), at(g.sPLl, mm, s0), mm);
    cp(at(g.PRh, nn, s0), at(g.sPRh, nn, s0), nn);
    cp(at(g.PRl, nn, s0), at(g.sPRl, nn, s0), nn);
    if (f16_mode(bs)) {  // the step's fp16 copies of the installed roots
        to_f16(g.PLh, g.nb, s0, cnt, int64_t(mm), g.PL16, g.plscale, g.amax2, s, g.pln1, g.M);
        to_f16(g.PRh, g.nb, s0, cnt, int64_t(nn), g.PR16, g.prscale, g.amax2, s, g.prn1, g.N);
    }
    if (is_kl(bs)) std::fill(g.v_ok.begin() + s0, g.v_ok.begin() + s0 + cnt, uint8_t(0));
}

// Device-side install of a finished refresh (install_refresh precond.cpp:144-164).
void install_apply(asg_blockset* bs, Unit& u) {
    Group& g = bs->groups[size_t(u.group)];
    if (f32_refresh(bs) && is_soap(bs)) {
        install_soap_f32(bs, g, u.slot, 1);
        return;
    }
    cudaStream_t s = bs->main;
    const size_t mm = slabMM(g), nn = slabNN(g);
    if (!is_soap(bs)) {
        install_roots(bs, g, u.slot, 1);
        return;
    }
    // SOAP: rot = Q_new^T Q_old per side; M <- rot_L M rot_R^T,
    // V <- (rot_L o rot_L) V (rot_R o rot_R)^T; swap bases.
    const int m = g.m, n = g.n;
    const size_t dm = size_t(m) * m, dn = size_t(n) * n, mnd = size_t(m) * n, MN = slabMN(g);
    double* qLn = at(g.sQL64, dm, u.slot);
    double* qLo = at(g.QL64, dm, u.slot);
    double* qRn = at(g.sQR64, dn, u.slot);
    double* qRo = at(g.QR64, dn, u.slot);
    launch_dgemm(true, false, m, m, m, 1.0, qLn, m, 0, qLo, m, 0, 0.0, bs->iw_rotL, m, 0, 1, s);
    launch_dgemm(true, false, n, n, n, 1.0, qRn, n, 0, qRo, n, 0, 0.0, bs->iw_rotR, n, 0, 1, s);
    for (int which = 0; which < 2; ++which) {
        float* mom = at(which == 0 ? g.mom_m : g.mom_v, MN, u.slot);
        const double* rl = bs->iw_rotL;
        const double* rr = bs->iw_rotR;
        if (which == 1) {
            launch_square_f64(bs->iw_rotL, bs->iw_sq, int64_t(dm), s);
            rl = bs->iw_sq;
        }
        launch_f32_to_f64(mom, 1, m, n, g.M, g.N, bs->iw_a, s);
        launch_dgemm(false, false, m, n, m, 1.0, rl, m, 0, bs->iw_a, n, 0, 0.0, bs->iw_b, n, 0, 1, s);
        if (which == 1) {
            // rot_R o rot_R into iw_a's spare? reuse rotR in place after squaring
            launch_square_f64(bs->iw_rotR, bs->iw_rotR, int64_t(dn), s);
            rr = bs->iw_rotR;
        }
        launch_dgemm(false, true, m, n, n, 1.0, bs->iw_b, n, 0, rr, n, 0, 0.0, bs->iw_a, n, 0, 1, s);
        launch_f64_to_f32(bs->iw_a, 1, m, n, mom, g.M, g.N, s);
    }
    (void)mnd;
    CK(cudaMemcpyAsync(qLo, qLn, dm * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(qRo, qRn, dn * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(at(g.valsL, size_t(m), u.slot), at(g.svalsL, size_t(m), u.slot), size_t(m) * 8,
                       cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(at(g.valsR, size_t(n), u.slot), at(g.svalsR, size_t(n), u.slot), size_t(n) * 8,
                       cudaMemcpyDeviceToDevice, s));
    launch_f64_to_split(qLo, 1, m, g.M, false, at(g.QLh, mm, u.slot), at(g.QLl, mm, u.slot), at(g.QLTh, mm, u.slot),
                        at(g.QLTl, mm, u.slot), s);
    launch_f64_to_split(qRo, 1, n, g.N, false, at(g.QRh, nn, u.slot), at(g.QRl, nn, u.slot), at(g.QRTh, nn, u.slot),
                        at(g.QRTl, nn, u.slot), s);
}

// ShadowScheduler::install (asyncsched.cpp:144-189): bookkeeping now (so the
// simulated clock and trace follow the reference's per-block order), device
// work deferred to run_deferred_installs().
void sched_install(asg_blockset* bs, int idx, int64_t step) {
    Unit& u = bs->units[size_t(idx)];
    bs->stats.completed += 1;
    emit(bs, u.dispatch_step, ASG_EV_JOB_START, idx, u.version, u.dispatch_sim);
    emit(bs, step, ASG_EV_JOB_DONE, idx, u.version, u.completion_sim);
    bs->deferred_installs.push_back(idx);
    u.version += 1;
    u.last_refresh_step = step;
    bs->now_us += bs->sc.install_cost_us;
    u.fresh.installed_version = u.version;
    u.fresh.last_install_step = step;
    u.fresh.installed_snapshot_step = u.dispatch_step;
    u.fresh.dispatch_step_of_pending = -1;
    u.pending = false;
    if (bs->store) emit(bs, step, ASG_EV_PREFETCH, idx, u.version, bs->now_us);  // asyncsched.cpp:183
    emit(bs, step, ASG_EV_INSTALL, idx, u.version, bs->now_us);
    bs->stats.installed += 1;
}

// F3 write-back (ShadowScheduler::install asyncsched.cpp:164-184): the
// refreshed inverse state (Shampoo / KL roots, SOAP bases) of each installed
// block goes to the store's Host tier (pinned) as it lives in HBM -- the
// padded fp32 (hi | lo) slabs, or the fp64 basis of the F64 refresh -- and is
// prefetched back toward Hot; ForwardPost drains it (asg_on_hook).
std::string unit_id(const asg_blockset* bs, int i);
void store_write_back(asg_blockset* bs, const std::vector<int>& todo) {
    CK(cudaStreamSynchronize(bs->main));  // the installs above are complete
    for (int idx : todo) {
        const Unit& u = bs->units[size_t(idx)];
        Group& g = bs->groups[size_t(u.group)];
        const std::string id = unit_id(bs, idx);
        for (int side = 0; side < 2; ++side) {
            const bool left = side == 0;
            const int32_t role = is_soap(bs) ? (left ? ASG_ROLE_BASIS_L : ASG_ROLE_BASIS_R)
                                             : (left ? ASG_ROLE_INV_L : ASG_ROLE_INV_R);
            const int d = left ? g.m : g.n, D = left ? g.M : g.N;
            const size_t DD = size_t(D) * D;
            const void* src = nullptr;
            uint64_t bytes = 0;
            if (is_soap(bs) && g.QL64) {  // F64 refresh: the fp64 basis itself
                src = at(left ? g.QL64 : g.QR64, size_t(d) * d, u.slot);
                bytes = uint64_t(d) * d * 8;
            } else {
                const float* hi = is_soap(bs) ? at(left ? g.QLh : g.QRh, DD, u.slot) : at(left ? g.PLh : g.PRh, DD, u.slot);
                const float* lo = is_soap(bs) ? at(left ? g.QLl : g.QRl, DD, u.slot) : at(left ? g.PLl : g.PRl, DD, u.slot);
                CK(cudaMemcpyAsync(bs->store_stage, hi, DD * 4, cudaMemcpyDeviceToDevice, bs->main));
                bytes = DD * 4;
                if (lo) {
                    CK(cudaMemcpyAsync(bs->store_stage + DD, lo, DD * 4, cudaMemcpyDeviceToDevice, bs->main));
                    bytes += DD * 4;
                }
                CK(cudaStreamSynchronize(bs->main));
                src = bs->store_stage;
            }
            int rc = asg_tier_put_device(bs->store, id.c_str(), role, src, bytes, ASG_TIER_HOST, nullptr);
            if (rc == ASG_OK) rc = asg_tier_prefetch(bs->store, id.c_str(), role, ASG_TIER_HOT, nullptr);
            if (rc != ASG_OK) throw Fail{rc, asg_last_error()};
            bs->queued_prefetches.push_back({id, role, idx, u.last_refresh_step});
        }
    }
}

// Launches every outstanding refresh as one batch, then performs the deferred
// device installs in decision order (main stream, before the update).
void run_deferred_installs(asg_blockset* bs) {
    launch_refreshes(bs);
    std::vector<int> todo;
    todo.swap(bs->deferred_installs);
    const bool host_wait = bs->sc.install_mode != ASG_INSTALL_EVENT;
    for (int idx : todo) install_wait(bs, bs->units[size_t(idx)], host_wait);
    if (f32_refresh(bs) && is_soap(bs)) {
        // batched: contiguous slot runs of one group, in workspace-sized chunks.
        // Blocks whose refresh left J = I on both sides (warm, nothing to rotate)
        // only take the new eigenvalues: basis and moments are unchanged.
        std::vector<std::pair<int, int>> gs, triv;
        for (int idx : todo) {
            const Unit& u = bs->units[size_t(idx)];
            const Group& g = bs->groups[size_t(u.group)];
            const bool trivial = g.h_identL && g.h_identL[u.slot] && g.h_identR[u.slot];
            (trivial ? triv : gs).emplace_back(u.group, u.slot);
        }
        std::sort(triv.begin(), triv.end());
        for (size_t i = 0; i < triv.size();) {
            size_t j = i + 1;
            while (j < triv.size() && triv[j].first == triv[i].first && triv[j].second == triv[j - 1].second + 1) ++j;
            Group& g = bs->groups[size_t(triv[i].first)];
            const int s0 = triv[i].second, cnt = int(j - i);
            CK(cudaMemcpyAsync(at(g.valsL, size_t(g.m), s0), at(g.svalsL, size_t(g.m), s0), size_t(cnt) * g.m * 8,
                               cudaMemcpyDeviceToDevice, bs->main));
            CK(cudaMemcpyAsync(at(g.valsR, size_t(g.n), s0), at(g.svalsR, size_t(g.n), s0), size_t(cnt) * g.n * 8,
                               cudaMemcpyDeviceToDevice, bs->main));
            i = j;
        }
        std::sort(gs.begin(), gs.end());
        size_t i = 0;
        while (i < gs.size()) {
            size_t j = i + 1;
            while (j < gs.size() && gs[j].first == gs[i].first && gs[j].second == gs[j - 1].second + 1 &&
                   int(j - i) < bs->ws_chunk)
                ++j;
            install_soap_f32(bs, bs->groups[size_t(gs[i].first)], gs[i].second, int(j - i));
            i = j;
        }
    } else if (!is_soap(bs)) {
        // roots: contiguous slot runs of one group, one copy per array per run
        std::vector<std::pair<int, int>> gs;
        for (int idx : todo) gs.emplace_back(bs->units[size_t(idx)].group, bs->units[size_t(idx)].slot);
        std::sort(gs.begin(), gs.end());
        for (size_t i = 0; i < gs.size();) {
            size_t j = i + 1;
            while (j < gs.size() && gs[j].first == gs[i].first && gs[j].second == gs[j - 1].second + 1) ++j;
            install_roots(bs, bs->groups[size_t(gs[i].first)], gs[i].second, int(j - i));
            i = j;
        }
    } else {
        for (int idx : todo) install_apply(bs, bs->units[size_t(idx)]);
    }
    for (int idx : todo) bs->units[size_t(idx)].launched = false;
    if (bs->store && !todo.empty()) store_write_back(bs, todo);
}

void install_device(asg_blockset* bs, Unit& u) {
    install_wait(bs, u, true);
    install_apply(bs, u);
}

// maybe_dispatch (asyncsched.cpp:108-142), host bookkeeping only.
bool sched_dispatch(asg_blockset* bs, int idx, int64_t step) {
    Unit& u = bs->units[size_t(idx)];
    if (step % bs->sc.pf != 0) return false;
    if (u.pending) {
        bs->stats.coalesced += 1;
        return false;
    }
    double cost = bs->sc.inject_job_delay_steps;
    if (bs->sc.inject_job_delay_jitter_steps > 0.0) {
        std::uniform_real_distribution<double> dist(0.0, bs->sc.inject_job_delay_jitter_steps);
        cost += dist(bs->jitter);
    }
    u.pending = true;
    u.launched = false;
    u.needs_launch = true;
    u.warm_start = u.version > 0;  // before this job's own install bookkeeping
    u.dispatch_step = step;
    u.dispatch_sim = bs->now_us;
    u.completion_sim = bs->now_us + cost * bs->sc.step_compute_us;
    emit(bs, step, ASG_EV_DISPATCH, idx, u.version, bs->now_us);
    u.has_fresh = true;
    u.fresh.dispatch_step_of_pending = step;
    bs->stats.dispatched += 1;
    return true;
}

// staleness_barrier (asyncsched.cpp:191-221).
double sched_barrier(asg_blockset* bs, int idx, int64_t step) {
    Unit& u = bs->units[size_t(idx)];
    if (!u.pending) return 0.0;
    const int64_t age = step - u.dispatch_step;
    const bool stale_consumer =
        u.version > 0 && step - u.fresh.installed_snapshot_step > (bs->sc.staleness_S + 1) * bs->sc.pf;
    const bool wait = bs->sc.staleness_S == 0 || age > bs->sc.staleness_S || stale_consumer;
    if (!wait) return 0.0;
    double waited;
    const double now = bs->now_us;
    if (bs->sc.install_mode == ASG_INSTALL_EVENT) {
        // the main stream waits on the refresh event; the host does not block.
        // The device-side wait is measured and added to wait_total_us when the
        // install resolves (resolve_deferred).
        waited = 0.0;
    } else {
        waited = std::max(0.0, u.completion_sim - now);
    }
    emit(bs, step, ASG_EV_BARRIER_WAIT_BEGIN, idx, u.version, now);
    bs->now_us += waited;
    sched_install(bs, idx, step);
    emit(bs, step, ASG_EV_BARRIER_WAIT_END, idx, u.version, bs->now_us);
    bs->stats.barrier_waits += 1;
    bs->stats.wait_total_us += waited;
    return waited;
}

// BlockSpec::id (precond.cpp:64-67) with the reference harness's parameter
// names "w<index>" (harness.cpp:357).
std::string unit_id(const asg_blockset* bs, int i) {
    const asg_block_spec& sp = bs->units[size_t(i)].spec;
    return "w" + std::to_string(sp.param_index) + "[" + std::to_string(sp.row_begin) + ":" +
           std::to_string(sp.row_end) + "," + std::to_string(sp.col_begin) + ":" + std::to_string(sp.col_end) + "]";
}

// on_hook(StepEnd) (asyncsched.cpp:268-286).
void sched_step_end(asg_blockset* bs, int64_t step) {
    launch_refreshes(bs);
    std::vector<int> ready;
    for (size_t i = 0; i < bs->units.size(); ++i) {
        Unit& u = bs->units[i];
        if (!u.pending) continue;
        bool ok;
        if (bs->sc.install_mode == ASG_INSTALL_EVENT)
            ok = u.launched && cudaEventQuery(u.done) == cudaSuccess;
        else
            ok = u.completion_sim <= bs->now_us;
        if (ok) ready.push_back(int(i));
    }
    // installs in ascending block-id order (asyncsched.cpp:275-276: std::sort
    // of BlockSpec::id strings, "w<param>[r0:r1,c0:c1]" as the reference
    // harness names them, harness.cpp:357, precond.cpp:64-67)
    std::sort(ready.begin(), ready.end(), [&](int a, int b) { return unit_id(bs, a) < unit_id(bs, b); });
    for (int i : ready) sched_install(bs, i, step);
    run_deferred_installs(bs);
}

void check_owned_index(const asg_blockset* bs, int64_t idx) {
    if (idx < 0 || idx >= int64_t(bs->units.size())) throw Fail{ASG_ERR_INVALID_ARGUMENT, "block index out of range"};
}

void stage_host_grad(asg_blockset* bs, const Unit& u, const double* g, int64_t ld) {
    const int m = int(u.spec.row_end - u.spec.row_begin), n = int(u.spec.col_end - u.spec.col_begin);
    std::vector<float> buf(size_t(m) * n);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
            const double x = g[size_t(i) * ld + j];
            if (!std::isfinite(x)) throw Fail{ASG_ERR_NON_FINITE, "accumulate_factors: non-finite gradient"};
            buf[size_t(i) * n + j] = float(x);
        }
    h2d(bs->stage, buf.data(), buf.size() * 4, bs->main);
    BlockRef r{bs->stage, nullptr, n, m, n};
    h2d(bs->d_ref1, &r, sizeof(r), bs->main);
}

Group& owned_group(asg_blockset* bs, const Unit& u) {
    if (u.adamw || u.group < 0) throw Fail{ASG_ERR_INVALID_ARGUMENT, "block is not a preconditioned block owned by this rank"};
    return bs->groups[size_t(u.group)];
}

void prep_single(asg_blockset* bs, Group& g, const Unit& u) {
    const size_t mn = slabMN(g);
    if (!g.v_ok.empty()) g.v_ok[size_t(u.slot)] = 0;
    if (f16_mode(bs)) {
        const size_t o = size_t(u.slot) * mn, lo = size_t(g.nb) * mn;
        launch_prep_grad_f16(bs->d_ref1, 1, g.M, g.N, 1.f, g.amax2 + u.slot, g.G16 + o, g.G16 + lo + o, g.GT16 + o,
                             g.GT16 + lo + o, g.gscale + u.slot, bs->main);
        return;
    }
    launch_prep_grad(bs->d_ref1, 1, g.M, g.N, nullptr, 1.f, at(g.Gh, mn, u.slot), at(g.Gl, mn, u.slot),
                     at(g.GTh, mn, u.slot), at(g.GTl, mn, u.slot), bs->main);
}

void download_block(asg_blockset* bs, Group& g, double* out) {
    std::vector<float> buf(slabMN(g));
    CK(cudaStreamSynchronize(bs->main));
    CK(cudaMemcpy(buf.data(), bs->d_out1, buf.size() * 4, cudaMemcpyDeviceToHost));
    for (int i = 0; i < g.m; ++i)
        for (int j = 0; j < g.n; ++j) out[size_t(i) * g.n + j] = double(buf[size_t(i) * g.N + j]);
}

// The update's NonFinite flag (apply_update precond.cpp:248; adamw_step
// precond.cpp:231): set on the device by EPI_APPLY / AdamW (which leave the
// non-finite elements of theta unchanged), surfaced here once the stream has
// been synchronized.
void check_flag(asg_blockset* bs) {
    int f = 0;
    CK(cudaMemcpy(&f, bs->d_upd_flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (f) {
        CK(cudaMemset(bs->d_upd_flag, 0, sizeof(int)));
        throw Fail{ASG_ERR_NON_FINITE, "apply_update: non-finite update"};
    }
}

// Resolves EVENT-mode barrier installs whose refresh has completed: the
// refresh status (a failure surfaces here, at the next host sync after the
// install) and the main stream's device-side wait (stats.wait_total_us).
// blocking: wait for every outstanding one.
void resolve_deferred(asg_blockset* bs, bool blocking) {
    std::vector<asg_blockset::DeferredInstall> keep;
    int fail = ASG_OK;
    for (auto& d : bs->deferred_status) {
        if (!blocking && cudaEventQuery(d.ev_b) != cudaSuccess) {
            keep.push_back(d);
            continue;
        }
        CK(cudaEventSynchronize(d.ev_b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, d.ev_a, d.ev_b));
        bs->stats.wait_total_us += 1e3 * double(ms);
        const Unit& u = bs->units[size_t(d.unit)];
        const int st = bs->groups[size_t(u.group)].h_status[u.slot];
        if (st != ASG_OK && fail == ASG_OK) fail = st;
        cudaEventDestroy(d.ev_a);
        cudaEventDestroy(d.ev_b);
    }
    bs->deferred_status.swap(keep);
    if (fail != ASG_OK) throw Fail{fail, "refresh (installed at an earlier barrier) failed"};
}

}  // namespace
}  // namespace asg

// ============================================================================
// C-ABI
// ============================================================================
using namespace asg;

namespace asg {
// the message of asg_last_error() for entry points defined in other files (asg_tierstore.cu)
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace asg

extern "C" {

const char* asg_last_error(void) { return g_err.c_str(); }
int asg_api_version(void) { return ASG_API_VERSION; }

int asg_device_supported(int device) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 0;
    return prop.major == 10 && prop.minor == 0 ? 1 : 0;
}

int asg_optimizer_defaults(int32_t method, asg_optimizer_config* out) {
    return guard([&] {
        if (!out) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null output"};
        *out = defaults_for(method);
    });
}

int asg_optimizer_validate(const asg_optimizer_config* cfg) {
    return guard([&] {
        if (!cfg) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null config"};
        validate(*cfg);
    });
}

int asg_scheduler_defaults(asg_scheduler_config* out) {
    return guard([&] { *out = sched_defaults(); });
}

int asg_config_from_json(const char* text, asg_optimizer_config* opt, asg_scheduler_config* sched, int32_t* precision) {
    return guard([&] {
        if (!text || !opt || !sched) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        json::Value j;
        try {
            j = json::Parser(text).parse();
        } catch (const std::exception& e) {
            throw Fail{ASG_ERR_CONFIG_INVALID, e.what()};
        }
        asg_optimizer_config o = defaults_for(ASG_METHOD_ADAMW);
        asg_scheduler_config s = sched_defaults();
        int32_t prec = ASG_PREC_3XTF32;
        auto num = [&](const json::Value& v, const char* k, auto& out) {
            if (!v.has(k)) return;
            const json::Value& x = v.at(k);
            if (x.kind != json::Value::Number) throw Fail{ASG_ERR_CONFIG_INVALID, std::string("not a number: ") + k};
            out = static_cast<std::remove_reference_t<decltype(out)>>(x.num);
        };
        auto str = [&](const json::Value& v, const char* k) -> std::string {
            const json::Value& x = v.at(k);
            if (x.kind != json::Value::String) throw Fail{ASG_ERR_CONFIG_INVALID, std::string("not a string: ") + k};
            return x.str;
        };
        if (j.has("optimizer")) {  // config.cpp:124-139
            const json::Value& v = j.at("optimizer");
            if (v.has("method")) o = defaults_for(method_from_string(str(v, "method")));
            num(v, "lr", o.lr);
            num(v, "beta1", o.beta1);
            num(v, "beta2", o.beta2);
            num(v, "eps", o.eps);
            num(v, "weight_decay", o.weight_decay);
            num(v, "precondition_frequency", o.precondition_frequency);
            if (v.has("accumulation")) {
                const std::string a = str(v, "accumulation");
                if (a == "Sum") o.accumulation = ASG_ACCUM_SUM;
                else if (a == "EMA") o.accumulation = ASG_ACCUM_EMA;
                else throw Fail{ASG_ERR_CONFIG_INVALID, "unknown accumulation mode: " + a};
            }
            num(v, "damping", o.damping);
            num(v, "block_dim_limit", o.block_dim_limit);
        }
        s.pf = o.precondition_frequency;  // config.cpp:140
        if (j.has("async")) {             // config.cpp:141-149
            const json::Value& a = j.at("async");
            num(a, "staleness_S", s.staleness_S);
            num(a, "pf", s.pf);
            num(a, "pool_size", s.pool_size);
            num(a, "inject_job_delay_steps", s.inject_job_delay_steps);
            num(a, "inject_job_delay_jitter_steps", s.inject_job_delay_jitter_steps);
            num(a, "drain_budget", s.drain_budget);
        }
        if (j.has("sim")) {  // config.cpp:193-202
            num(j.at("sim"), "step_compute_us", s.step_compute_us);
            num(j.at("sim"), "install_cost_us", s.install_cost_us);
        } else {
            s.install_cost_us = 10.0;  // SimCostConfig default (harness.hpp:51-54)
        }
        if (j.has("gpu")) {
            const json::Value& g = j.at("gpu");
            if (g.has("precision")) {
                const std::string p = str(g, "precision");
                if (p == "3xtf32") prec = ASG_PREC_3XTF32;
                else if (p == "3xtf32_smem") prec = ASG_PREC_3XTF32_SMEM;
                else if (p == "3xf16") prec = ASG_PREC_3XF16;
                else if (p == "tf32") prec = ASG_PREC_TF32;
                else throw Fail{ASG_ERR_CONFIG_INVALID, "unknown precision: " + p};
            }
            if (g.has("refresh")) {
                const std::string r = str(g, "refresh");
                if (r == "f64") s.refresh_mode = ASG_REFRESH_F64;
                else if (r == "f32") s.refresh_mode = ASG_REFRESH_F32;
                else if (r == "newton") s.refresh_mode = ASG_REFRESH_NEWTON;
                else throw Fail{ASG_ERR_CONFIG_INVALID, "unknown refresh: " + r};
            }
            if (g.has("install_mode")) {
                const std::string m = str(g, "install_mode");
                if (m == "sim_clock") s.install_mode = ASG_INSTALL_SIM_CLOCK;
                else if (m == "event") s.install_mode = ASG_INSTALL_EVENT;
                else throw Fail{ASG_ERR_CONFIG_INVALID, "unknown install_mode: " + m};
            }
        }
        validate(o);  // config.cpp:40-43
        if (s.pf != o.precondition_frequency)
            throw Fail{ASG_ERR_CONFIG_INVALID, "async.pf must equal optimizer.precondition_frequency"};
        if (s.staleness_S < 0) throw Fail{ASG_ERR_CONFIG_INVALID, "staleness_S must be >= 0"};
        *opt = o;
        *sched = s;
        if (precision) *precision = prec;
    });
}

int asg_partition_param(int64_t param_index, int64_t rows, int64_t cols, int64_t limit, asg_block_spec* out,
                        int64_t capacity, int64_t* count) {
    return guard([&] {
        if (limit < 1) throw Fail{ASG_ERR_CONFIG_INVALID, "partition_param: limit must be >= 1"};
        if (rows < 1 || cols < 1) throw Fail{ASG_ERR_SHAPE_MISMATCH, "partition_param: empty parameter"};
        int64_t k = 0;
        for (int64_t r = 0; r < rows; r += limit)
            for (int64_t c = 0; c < cols; c += limit) {
                if (out && k < capacity)
                    out[k] = asg_block_spec{param_index, r, std::min(rows, r + limit), c, std::min(cols, c + limit), limit};
                ++k;
            }
        if (count) *count = k;
    });
}

int asg_blockset_create(int device, const asg_optimizer_config* opt, const asg_scheduler_config* sched,
                        const asg_param_desc* params, int64_t n_params, int32_t precision, int32_t rank, int32_t world,
                        uint64_t seed, asg_blockset** out) {
    asg_blockset* bs = nullptr;
    int rc = guard([&] {
        if (!opt || !sched || !out || (n_params > 0 && !params)) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        validate(*opt);
        if (sched->staleness_S < 0) throw Fail{ASG_ERR_CONFIG_INVALID, "staleness_S must be >= 0"};
        if (sched->pf < 1) throw Fail{ASG_ERR_CONFIG_INVALID, "pf must be >= 1"};
        if (sched->refresh_mode != ASG_REFRESH_F64 && sched->refresh_mode != ASG_REFRESH_F32 &&
            sched->refresh_mode != ASG_REFRESH_NEWTON)
            throw Fail{ASG_ERR_CONFIG_INVALID, "unknown refresh_mode"};
        if (sched->pf != opt->precondition_frequency)
            throw Fail{ASG_ERR_CONFIG_INVALID, "async.pf must equal optimizer.precondition_frequency"};
        if (world < 1 || rank < 0 || rank >= world) throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad rank/world"};
        if (precision != ASG_PREC_3XTF32 && precision != ASG_PREC_TF32 && precision != ASG_PREC_3XTF32_SMEM &&
            precision != ASG_PREC_3XF16)
            throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad precision"};
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
            throw Fail{ASG_ERR_UNSUPPORTED, "no CUDA device " + std::to_string(device)};
        if (!asg_device_supported(device))
            throw Fail{ASG_ERR_UNSUPPORTED, "device is not sm_100 (B200); this library has no other code path"};
        CK(cudaSetDevice(device));
        bs = new asg_blockset();
        bs->device = device;
        bs->opt = *opt;
        bs->sc = *sched;
        bs->precision = precision;
        bs->rank = rank;
        bs->world = world;
        bs->jitter.seed(seed * 0x9e3779b97f4a7c15ull + 0x2545f4914f6cdd1dull);  // asyncsched.cpp:248
        bs->params.assign(params, params + n_params);
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        bs->num_sms = prop.multiProcessorCount;
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&bs->main, cudaStreamNonBlocking, hi));
        static const bool same_prio = getenv("ASG_SIDE_SAME_PRIORITY") != nullptr;  // diagnostics
        CK(cudaStreamCreateWithPriority(&bs->side, cudaStreamNonBlocking, same_prio ? hi : lo));
        CK(cudaStreamCreateWithPriority(&bs->side2, cudaStreamNonBlocking, same_prio ? hi : lo));
        bs->own_main = true;
        for (int k = 0; k < asg_blockset::kGroupStreams; ++k) {
            CK(cudaStreamCreateWithPriority(&bs->gstream[k], cudaStreamNonBlocking, hi));
            CK(cudaEventCreateWithFlags(&bs->gjoin[k], cudaEventDisableTiming));
        }
        CK(cudaEventCreateWithFlags(&bs->gfork, cudaEventDisableTiming));
        bs->fp64_jacobi = getenv("ASG_F32_FP64_JACOBI") != nullptr;
        CK(cudaEventCreateWithFlags(&bs->ev_snap, cudaEventDisableTiming));
        build_units(bs);
        build_groups(bs);
        for (Group& g : bs->groups) alloc_group(bs, g);
        const size_t before_ws = bs->alloc_bytes;
        alloc_workspace(bs);
        bs->workspace_bytes = bs->alloc_bytes - before_ws;
        for (Unit& u : bs->units) {
            CK(cudaEventCreateWithFlags(&u.done, cudaEventDisableTiming));
            if (u.adamw && u.owner == rank) {
                const size_t n = size_t(u.spec.row_end - u.spec.row_begin) * size_t(u.spec.col_end - u.spec.col_begin);
                u.am = dalloc<float>(bs, n);
                u.av = dalloc<float>(bs, n);
                CK(cudaMemsetAsync(u.am, 0, n * 4, bs->main));
                CK(cudaMemsetAsync(u.av, 0, n * 4, bs->main));
            }
        }
        build_adam_table(bs);
        build_sq_table(bs);
        bs->d_flag = dalloc<int>(bs, 1);
        bs->d_upd_flag = dalloc<int>(bs, 1);
        bs->h_upd_flag = halloc<int>(bs, 1);
        bs->d_sqnorm = dalloc<double>(bs, 1);
        bs->d_scale = dalloc<float>(bs, 1);
        CK(cudaMemsetAsync(bs->d_flag, 0, sizeof(int), bs->main));
        CK(cudaMemsetAsync(bs->d_upd_flag, 0, sizeof(int), bs->main));
        size_t stage = 0;
        for (const Group& g : bs->groups) stage = std::max(stage, slabMN(g));
        bs->stage_elems = stage;
        bs->stage = dalloc<float>(bs, std::max<size_t>(stage, 1));
        bs->d_out1 = dalloc<float>(bs, std::max<size_t>(stage, 1));
        bs->d_ref1 = dalloc<BlockRef>(bs, 1);
        bs->d_apply1 = dalloc<ApplyEntry>(bs, 1);
        build_owner_layout(bs);
        CK(cudaStreamSynchronize(bs->main));
        CK(cudaGetLastError());
        *out = bs;
    });
    if (rc != ASG_OK && bs) {
        std::string keep = g_err;
        asg_blockset_destroy(bs);
        g_err = keep;
    }
    return rc;
}

int asg_blockset_destroy(asg_blockset* bs) {
    if (!bs) return ASG_OK;
    cudaSetDevice(bs->device);
    if (bs->main) cudaStreamSynchronize(bs->main);
    if (bs->side) cudaStreamSynchronize(bs->side);
    if (bs->side2) cudaStreamSynchronize(bs->side2);
    for (int k = 0; k < asg_blockset::kGroupStreams; ++k) {
        if (bs->gstream[k]) {
            cudaStreamSynchronize(bs->gstream[k]);
            cudaStreamDestroy(bs->gstream[k]);
        }
        if (bs->gjoin[k]) cudaEventDestroy(bs->gjoin[k]);
    }
    if (bs->gfork) cudaEventDestroy(bs->gfork);
    for (auto& u : bs->units)
        if (u.done) cudaEventDestroy(u.done);
    if (bs->ev_snap) cudaEventDestroy(bs->ev_snap);
    for (auto& e : bs->prof_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    for (auto& h : bs->prof_hbm) {
        cudaEventDestroy(h.e0);
        cudaEventDestroy(h.e1);
    }
    for (void* p : bs->allocs) cudaFree(p);
    for (void* p : bs->host_allocs) cudaFreeHost(p);
    for (cudaEvent_t e : bs->ag_events) cudaEventDestroy(e);
    if (bs->ag_done) cudaEventDestroy(bs->ag_done);
    if (bs->comm_stream) cudaStreamDestroy(bs->comm_stream);
    if (bs->own_main && bs->main) cudaStreamDestroy(bs->main);
    if (bs->side) cudaStreamDestroy(bs->side);
    if (bs->side2) cudaStreamDestroy(bs->side2);
    delete bs;
    return ASG_OK;
}

int asg_blockset_bind_params(asg_blockset* bs, const asg_param_desc* params, int64_t n_params) {
    return guard([&] {
        if (!bs || !params || n_params != int64_t(bs->params.size())) throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad params"};
        for (int64_t i = 0; i < n_params; ++i)
            if (params[i].rows != bs->params[size_t(i)].rows || params[i].cols != bs->params[size_t(i)].cols)
                throw Fail{ASG_ERR_SHAPE_MISMATCH, "bind_params: shape changed"};
        CK(cudaSetDevice(bs->device));
        CK(cudaStreamSynchronize(bs->main));
        bs->params.assign(params, params + n_params);
        for (Group& g : bs->groups) bind_group_tables(bs, g);
        build_adam_table(bs);
        build_sq_table(bs);
        build_owner_layout(bs);
        if (!bs->buckets.empty()) build_buckets(bs, bs->buckets_per_shape);
    });
}

int asg_blockset_num_blocks(const asg_blockset* bs, int64_t* n) {
    return guard([&] {
        if (!bs || !n) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        *n = int64_t(bs->units.size());
    });
}

int asg_blockset_block_info(const asg_blockset* bs, int64_t idx, asg_block_info* out) {
    return guard([&] {
        if (!bs || !out) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        check_owned_index(bs, idx);
        const Unit& u = bs->units[size_t(idx)];
        out->spec = u.spec;
        out->version = u.version;
        out->last_refresh_step = u.last_refresh_step;
        out->moment_steps = u.moment_steps;
        out->owner_rank = u.owner;
        out->use_adamw = u.adamw ? 1 : 0;
    });
}

int asg_blockset_state_bytes(const asg_blockset* bs, uint64_t* bytes) {
    return guard([&] { *bytes = bs->alloc_bytes - bs->workspace_bytes; });
}

int asg_blockset_workspace_bytes(const asg_blockset* bs, uint64_t* bytes) {
    return guard([&] { *bytes = bs->workspace_bytes; });
}

int asg_blockset_stream(const asg_blockset* bs, void** stream) {
    return guard([&] { *stream = bs->main; });
}

int asg_grad_sqnorm(asg_blockset* bs, void* stream, double* sqnorm, int32_t* nonfinite) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        CK(cudaMemsetAsync(bs->d_sqnorm, 0, sizeof(double), s));
        CK(cudaMemsetAsync(bs->d_flag, 0, sizeof(int), s));
        double elems = 0.0;
        for (const asg_param_desc& d : bs->params) elems += d.grad ? double(d.rows) * double(d.cols) : 0.0;
        hbm_launch(bs, s, ASG_HBM_SQNORM, 4.0 * elems, [&] {
            launch_sqnorm_multi(bs->d_sq, bs->n_sq, bs->d_sqnorm, bs->d_flag, s);  // every parameter, one launch
        });
        double v = 0.0;
        int f = 0, fu = 0;
        CK(cudaMemcpyAsync(&v, bs->d_sqnorm, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&f, bs->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        // the previous step's update flag (s is ordered after the step that wrote it)
        CK(cudaMemcpyAsync(&fu, bs->d_upd_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaMemsetAsync(bs->d_flag, 0, sizeof(int), s));
        if (sqnorm) *sqnorm = v;
        if (nonfinite) *nonfinite = f;
        resolve_deferred(bs, false);
        if (fu) {
            CK(cudaMemsetAsync(bs->d_upd_flag, 0, sizeof(int), s));
            throw Fail{ASG_ERR_NON_FINITE, "apply_update: the previous step's update was non-finite "
                                           "(those elements of theta were left unchanged)"};
        }
    });
}

int asg_accumulate(asg_blockset* bs, double clip_scale, void* stream) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        if (s != bs->main) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CK(cudaEventRecord(e, s));
            CK(cudaStreamWaitEvent(bs->main, e, 0));
            CK(cudaEventDestroy(e));
        }
        accumulate_impl(bs, clip_scale);
        CK(cudaGetLastError());
    });
}

int asg_maybe_dispatch(asg_blockset* bs, int64_t step, int64_t* n_dispatched) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        int64_t n = 0;
        for (size_t i = 0; i < bs->units.size(); ++i) {
            const Unit& u = bs->units[i];
            if (u.adamw || u.owner != bs->rank) continue;
            n += sched_dispatch(bs, int(i), step) ? 1 : 0;
        }
        launch_refreshes(bs);
        if (n_dispatched) *n_dispatched = n;
    });
}

int asg_staleness_barrier(asg_blockset* bs, int64_t step, double* waited_us) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        double w = 0.0;
        for (size_t i = 0; i < bs->units.size(); ++i) {
            const Unit& u = bs->units[i];
            if (u.adamw || u.owner != bs->rank) continue;
            w += sched_barrier(bs, int(i), step);
        }
        run_deferred_installs(bs);
        if (waited_us) *waited_us = w;
    });
}

namespace {
void adamw_impl(asg_blockset* bs, double clip_scale, float lr_eff, cudaStream_t as);

void precondition_apply_impl(asg_blockset* bs, double clip_scale, double lr_scale) {
    const float lr_eff = float(bs->opt.lr * lr_scale);
    for (size_t gi = 0; gi < bs->groups.size(); ++gi) {
        Group& g = bs->groups[gi];
        if (is_soap(bs)) {
            int64_t ms = -1;
            for (int ui : g.units) {
                Unit& u = bs->units[size_t(ui)];
                u.moment_steps += 1;
                if (ms >= 0 && u.moment_steps != ms) throw Fail{ASG_ERR_AUDIT, "SOAP moment steps diverged within a group"};
                ms = u.moment_steps;
            }
        }
    }
    if (bs->ag_comm) {
        // fused all-gather: the update runs bucket by bucket on the main stream;
        // bucket b's all-gather (comm stream) overlaps the update of b+1
        ncclComm_t comm = static_cast<ncclComm_t>(bs->ag_comm);
        CK(cudaEventRecord(bs->ag_done, bs->main));  // the comm stream starts after this step's earlier work
        CK(cudaStreamWaitEvent(bs->comm_stream, bs->ag_done, 0));
        bool adam_done = false;
        for (size_t i = 0; i < bs->buckets.size(); ++i) {
            const auto& b = bs->buckets[i];
            if (b.adamw) {
                if (!adam_done) adamw_impl(bs, clip_scale, lr_eff, bs->main);
                adam_done = true;
            } else if (b.cnt > 0) {
                Group& g = bs->groups[size_t(b.group)];
                group_update(bs, g, b.s0, b.cnt, EPI_APPLY, lr_eff, g.d_apply + b.s0, nullptr, bs->main);
            }
            CK(cudaEventRecord(bs->ag_events[i], bs->main));
            CK(cudaStreamWaitEvent(bs->comm_stream, bs->ag_events[i], 0));
            bucket_exchange(bs, b, comm, bs->comm_stream);
        }
        if (!adam_done) adamw_impl(bs, clip_scale, lr_eff, bs->main);
        CK(cudaEventRecord(bs->ag_done, bs->comm_stream));
        CK(cudaStreamWaitEvent(bs->main, bs->ag_done, 0));
        CK(cudaGetLastError());
        return;
    }
    const int k = fork_groups(bs);
    for (size_t gi = 0; gi < bs->groups.size(); ++gi) {
        Group& g = bs->groups[gi];
        group_update(bs, g, 0, g.nb, EPI_APPLY, lr_eff, g.d_apply, nullptr, stream_for(bs, k, int(gi)));
    }
    cudaStream_t as = stream_for(bs, k, int(bs->groups.size()));  // AdamW on the least loaded group stream
    adamw_impl(bs, clip_scale, lr_eff, as);
    join_groups(bs, k);
    CK(cudaGetLastError());
}

// AdamW for every owned 1-D / degenerate parameter in one launch (they step together)
void adamw_impl(asg_blockset* bs, double clip_scale, float lr_eff, cudaStream_t as) {
    int64_t t_adam = 0;
    for (Unit& u : bs->units) {
        if (!u.adamw || u.owner != bs->rank) continue;
        u.adam_t += 1;
        t_adam = u.adam_t;
    }
    if (bs->n_adam > 0) {
        const double t = double(t_adam);
        double elems = 0.0;
        for (const Unit& u : bs->units)
            if (u.adamw && u.owner == bs->rank)
                elems += double(u.spec.row_end - u.spec.row_begin) * double(u.spec.col_end - u.spec.col_begin);
        hbm_launch(bs, as, ASG_HBM_ADAMW, 28.0 * elems, [&] {  // theta r/w, g r, m r/w, v r/w
            launch_adamw_multi(bs->d_adam, bs->n_adam, bs->adam_max_elems, float(clip_scale), float(bs->opt.beta1),
                               float(bs->opt.beta2), float(1.0 / (1.0 - std::pow(bs->opt.beta1, t))),
                               float(1.0 / (1.0 - std::pow(bs->opt.beta2, t))), float(bs->opt.eps), lr_eff,
                               float(bs->opt.weight_decay), bs->d_upd_flag, as);
        });
    }
}
}  // namespace

int asg_precondition_apply(asg_blockset* bs, int64_t step, double clip_scale, double lr_scale, void* stream) {
    (void)step;
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        precondition_apply_impl(bs, clip_scale, lr_scale);
        if (stream && static_cast<cudaStream_t>(stream) != bs->main) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CK(cudaEventRecord(e, bs->main));
            CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), e, 0));
            CK(cudaEventDestroy(e));
        }
    });
}

int asg_step_end(asg_blockset* bs, int64_t step) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        sched_step_end(bs, step);
        if (bs->store) {  // asyncsched.cpp:284
            const int rc = asg_tier_advance_step(bs->store, step);
            if (rc != ASG_OK) throw Fail{rc, asg_last_error()};
        }
    });
}

// Synthetic gradients of this rank's units (benchmark input):
// unit u's gradient slice <- N(0, 1/cols(param)) i.i.d., Philox keyed (seed, step, u).
int asg_synth_gradients(asg_blockset* bs, uint64_t seed, int64_t step, void* stream) {
    return guard([&] {
        if (!bs) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null blockset"};
        CK(cudaSetDevice(bs->device));
        if (!bs->d_synth) {
            std::vector<SynthBlock> v;
            for (size_t i = 0; i < bs->units.size(); ++i) {
                const Unit& u = bs->units[i];
                if (u.owner != bs->rank) continue;
                const asg_param_desc& d = bs->params[size_t(u.spec.param_index)];
                if (!d.grad) continue;
                const int64_t r0 = u.spec.row_begin, r1 = u.spec.row_end, c0 = u.spec.col_begin, c1 = u.spec.col_end;
                SynthBlock b{const_cast<float*>(d.grad) + r0 * d.ld_grad + c0, d.ld_grad, int32_t(r1 - r0),
                             int32_t(c1 - c0), float(1.0 / std::sqrt(double(d.cols))), uint32_t(i)};
                bs->synth_rows = std::max(bs->synth_rows, int(b.rows));
                bs->synth_cols = std::max(bs->synth_cols, int(b.cols));
                v.push_back(b);
            }
            bs->n_synth = int(v.size());
            if (!v.empty()) {
                bs->d_synth = dalloc<SynthBlock>(bs, v.size());
                h2d(bs->d_synth, v.data(), v.size() * sizeof(SynthBlock), bs->main);
                CK(cudaStreamSynchronize(bs->main));
            }
        }
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        launch_synth_normal(bs->d_synth, bs->n_synth, bs->synth_rows, bs->synth_cols, seed, uint64_t(step), s);
        CK(cudaGetLastError());
    });
}

int asg_blockset_attach_store(asg_blockset* bs, asg_tierstore* store) {
    return guard([&] {
        if (!bs) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null blockset"};
        CK(cudaSetDevice(bs->device));
        bs->store = store;
        bs->queued_prefetches.clear();
        if (store && !bs->store_stage) {
            size_t mx = 0;
            for (const Group& g : bs->groups) mx = std::max({mx, size_t(g.M) * g.M, size_t(g.N) * g.N});
            bs->store_stage_floats = 2 * mx;
            if (mx) bs->store_stage = dalloc<float>(bs, bs->store_stage_floats);
        }
    });
}

// on_hook(ForwardPost / BackwardPre) asyncsched.cpp:223-267 (StepEnd is asg_step_end)
int asg_on_hook(asg_blockset* bs, int32_t kind, int64_t step) {
    return guard([&] {
        if (!bs) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null blockset"};
        if (kind == ASG_HOOK_STEP_END) {
            const int rc = asg_step_end(bs, step);
            if (rc != ASG_OK) throw Fail{rc, asg_last_error()};
            return;
        }
        if (!bs->store) return;
        auto ok = [](int rc) {
            if (rc != ASG_OK) throw Fail{rc, asg_last_error()};
        };
        if (kind == ASG_HOOK_FORWARD_POST) {
            // deterministic drain: only transfers enqueued before this step count,
            // and the (real) link time is waited out for them
            int budget = bs->sc.drain_budget;
            while (budget > 0 && !bs->queued_prefetches.empty() && bs->queued_prefetches.front().enqueue_step < step) {
                const asg_blockset::QueuedPrefetch q = bs->queued_prefetches.front();
                bs->queued_prefetches.pop_front();
                for (int spins = 0; spins < 200000; ++spins) {
                    int32_t n = 0;
                    ok(asg_tier_drain_ready(bs->store, bs->sc.drain_budget, &n));
                    asg_entry_view v{};
                    ok(asg_tier_inspect(bs->store, q.block_id.c_str(), q.role, &v));
                    if (!v.staged_pending && !v.staged_ready) break;
                    std::this_thread::sleep_for(std::chrono::microseconds(50));
                }
                const Unit& u = bs->units[size_t(q.unit)];
                emit(bs, step, ASG_EV_DRAIN, q.unit, u.fresh.installed_version, bs->now_us);
                budget -= 1;
            }
        } else if (kind == ASG_HOOK_BACKWARD_PRE) {
            for (size_t i = 0; i < bs->units.size(); ++i) {
                const Unit& u = bs->units[i];
                if (u.adamw || u.group < 0) continue;
                const std::string id = unit_id(bs, int(i));
                for (int side = 0; side < 2; ++side) {
                    const int32_t role = is_soap(bs) ? (side == 0 ? ASG_ROLE_BASIS_L : ASG_ROLE_BASIS_R)
                                                     : (side == 0 ? ASG_ROLE_INV_L : ASG_ROLE_INV_R);
                    int32_t has = 0;
                    ok(asg_tier_contains(bs->store, id.c_str(), role, &has));
                    if (!has) continue;
                    asg_entry_view v{};
                    ok(asg_tier_inspect(bs->store, id.c_str(), role, &v));
                    if (v.tier == ASG_TIER_COLD) {
                        ok(asg_tier_prefetch(bs->store, id.c_str(), role, ASG_TIER_HOST, nullptr));
                        bs->queued_prefetches.push_back({id, role, int(i), step});
                        emit(bs, step, ASG_EV_PREFETCH, int64_t(i), u.version, bs->now_us);
                    }
                }
            }
        } else {
            throw Fail{ASG_ERR_INVALID_ARGUMENT, "unknown hook kind"};
        }
    });
}

int asg_step(asg_blockset* bs, int64_t step, double clip_scale, double lr_scale, void* stream) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        if (s != bs->main) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CK(cudaEventRecord(e, s));
            CK(cudaStreamWaitEvent(bs->main, e, 0));
            CK(cudaEventDestroy(e));
        }
        static const bool host_timing = getenv("ASG_HOST_TIMING") != nullptr;  // diagnostics
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        accumulate_impl(bs, clip_scale);
        const auto t1 = clk::now();
        // per-block dispatch -> barrier in the reference's order (harness.cpp:452-454);
        // a barrier install launches any outstanding refresh first.
        for (size_t i = 0; i < bs->units.size(); ++i) {
            const Unit& u = bs->units[i];
            if (u.adamw || u.owner != bs->rank) continue;
            sched_dispatch(bs, int(i), step);
            sched_barrier(bs, int(i), step);
        }
        run_deferred_installs(bs);
        const auto t2 = clk::now();
        precondition_apply_impl(bs, clip_scale, lr_scale);
        const auto t3 = clk::now();
        sched_step_end(bs, step);
        const auto t4 = clk::now();
        if (host_timing) {
            auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            std::fprintf(stderr, "asg_step %lld host ms: accumulate %.2f dispatch/barrier/install %.2f update %.2f step_end %.2f\n",
                         (long long)step, ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
        }
        if (s != bs->main) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CK(cudaEventRecord(e, bs->main));
            CK(cudaStreamWaitEvent(s, e, 0));
            CK(cudaEventDestroy(e));
        }
    });
}

int asg_clock_advance(asg_blockset* bs, double us) {
    return guard([&] { bs->now_us += us; });
}

int asg_get_freshness(const asg_blockset* bs, int64_t idx, asg_freshness* out) {
    return guard([&] {
        check_owned_index(bs, idx);
        const Unit& u = bs->units[size_t(idx)];
        if (!u.has_fresh) throw Fail{ASG_ERR_MISSING_KEY, "asyncsched: no freshness record"};
        *out = u.fresh;
    });
}

int asg_get_stats(const asg_blockset* bs, asg_pool_stats* out) {
    return guard([&] {
        *out = bs->stats;
        int pending = 0;
        for (const Unit& u : bs->units) pending += u.pending ? 1 : 0;
        out->pending = pending;
        out->queue_depth = 0;
    });
}

int asg_get_events(const asg_blockset* bs, asg_event* out, int64_t capacity, int64_t* count) {
    return guard([&] {
        const int64_t n = int64_t(bs->events.size());
        for (int64_t i = 0; i < std::min(n, capacity); ++i) out[i] = bs->events[size_t(i)];
        if (count) *count = n;
    });
}

int asg_synchronize(asg_blockset* bs) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        CK(cudaStreamSynchronize(bs->main));
        sync_side(bs);
        resolve_deferred(bs, true);
        check_flag(bs);
    });
}

// ---- per-block parity entry points ------------------------------------------
int asg_block_read(asg_blockset* bs, int64_t idx, int32_t role, double* out, int64_t count) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        check_owned_index(bs, idx);
        const Unit& u = bs->units[size_t(idx)];
        Group& g = owned_group(bs, u);
        CK(cudaStreamSynchronize(bs->main));
        sync_side(bs);
        const int m = g.m, n = g.n;
        auto rd32 = [&](const float* base, size_t stride, int R, int Cc, int rows, int cols, const float* lo) {
            if (count < int64_t(rows) * cols) throw Fail{ASG_ERR_SHAPE_MISMATCH, "output too small"};
            if (!base) throw Fail{ASG_ERR_INVALID_ARGUMENT, "role not held by this method"};
            std::vector<float> h(size_t(R) * Cc), l;
            CK(cudaMemcpy(h.data(), base + stride * u.slot, h.size() * 4, cudaMemcpyDeviceToHost));
            if (lo) {
                l.resize(h.size());
                CK(cudaMemcpy(l.data(), lo + stride * u.slot, l.size() * 4, cudaMemcpyDeviceToHost));
            }
            for (int i = 0; i < rows; ++i)
                for (int j = 0; j < cols; ++j)
                    out[size_t(i) * cols + j] = double(h[size_t(i) * Cc + j]) + (lo ? double(l[size_t(i) * Cc + j]) : 0.0);
        };
        auto rd64 = [&](const double* base, size_t stride, size_t cnt) {
            if (count < int64_t(cnt)) throw Fail{ASG_ERR_SHAPE_MISMATCH, "output too small"};
            if (!base) throw Fail{ASG_ERR_INVALID_ARGUMENT, "role not held by this method"};
            CK(cudaMemcpy(out, base + stride * u.slot, cnt * 8, cudaMemcpyDeviceToHost));
        };
        switch (role) {
            case ASG_ROLE_FACTOR_L: rd32(g.L, slabMM(g), g.M, g.M, m, m, nullptr); break;
            case ASG_ROLE_FACTOR_R: rd32(g.R, slabNN(g), g.N, g.N, n, n, nullptr); break;
            case ASG_ROLE_INV_L: rd32(g.PLh, slabMM(g), g.M, g.M, m, m, g.PLl); break;
            case ASG_ROLE_INV_R: rd32(g.PRh, slabNN(g), g.N, g.N, n, n, g.PRl); break;
            case ASG_ROLE_KL_INV_L:
            case ASG_ROLE_KL_INV_R: {
                // F^-1 = (F^-1/2)^2 (not stored, group_stats): the installed root squared in fp64
                if (!is_kl(bs)) throw Fail{ASG_ERR_INVALID_ARGUMENT, "role not held by this method"};
                const bool left = role == ASG_ROLE_KL_INV_L;
                const int d = left ? m : n;
                if (count < int64_t(d) * d) throw Fail{ASG_ERR_SHAPE_MISMATCH, "output too small"};
                if (left)
                    rd32(g.PLh, slabMM(g), g.M, g.M, m, m, g.PLl);
                else
                    rd32(g.PRh, slabNN(g), g.N, g.N, n, n, g.PRl);
                const size_t dd = size_t(d) * d;
                h2d(bs->ws_out, out, dd * 8, bs->main);
                launch_dgemm(false, false, d, d, d, 1.0, bs->ws_out, d, 0, bs->ws_out, d, 0, 0.0, bs->ws_W, d, 0, 1,
                             bs->main);
                CK(cudaStreamSynchronize(bs->main));
                CK(cudaMemcpy(out, bs->ws_W, dd * 8, cudaMemcpyDeviceToHost));
                break;
            }
            case ASG_ROLE_BASIS_L:
                if (g.QL64) rd64(g.QL64, size_t(m) * m, size_t(m) * m);
                else rd32(g.QLh, slabMM(g), g.M, g.M, m, m, g.QLl);  // F32 refresh: split basis
                break;
            case ASG_ROLE_BASIS_R:
                if (g.QR64) rd64(g.QR64, size_t(n) * n, size_t(n) * n);
                else rd32(g.QRh, slabNN(g), g.N, g.N, n, n, g.QRl);
                break;
            case ASG_ROLE_EIGVALS_L: rd64(g.valsL, size_t(m), size_t(m)); break;
            case ASG_ROLE_EIGVALS_R: rd64(g.valsR, size_t(n), size_t(n)); break;
            case ASG_ROLE_ROTATED_M: rd32(g.mom_m, slabMN(g), g.M, g.N, m, n, nullptr); break;
            case ASG_ROLE_ROTATED_V: rd32(g.mom_v, slabMN(g), g.M, g.N, m, n, nullptr); break;
            default: throw Fail{ASG_ERR_INVALID_ARGUMENT, "unknown role"};
        }
    });
}

int asg_block_write(asg_blockset* bs, int64_t idx, int32_t role, const double* in, int64_t count) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        check_owned_index(bs, idx);
        const Unit& u = bs->units[size_t(idx)];
        Group& g = owned_group(bs, u);
        if (!g.v_ok.empty()) g.v_ok[size_t(u.slot)] = 0;  // roots may change: KL's cached V = P_L G is stale
        CK(cudaStreamSynchronize(bs->main));
        sync_side(bs);
        const int m = g.m, n = g.n;
        auto wr32 = [&](float* base, size_t stride, int R, int Cc, int rows, int cols, float* lo, float* hi_t, float* lo_t) {
            if (count < int64_t(rows) * cols) throw Fail{ASG_ERR_SHAPE_MISMATCH, "input too small"};
            if (!base) throw Fail{ASG_ERR_INVALID_ARGUMENT, "role not held by this method"};
            std::vector<double> buf(size_t(rows) * cols);
            std::memcpy(buf.data(), in, buf.size() * 8);
            double* d = bs->ws_out ? bs->ws_out : nullptr;
            if (!d || size_t(rows) * cols > size_t(bs->ws_n) * bs->ws_n) throw Fail{ASG_ERR_INVALID_ARGUMENT, "no staging space"};
            h2d(d, buf.data(), buf.size() * 8, bs->main);
            if (lo || hi_t) {
                launch_f64_to_split(d, 1, rows, R, false, base + stride * u.slot, lo ? lo + stride * u.slot : nullptr,
                                    hi_t ? hi_t + stride * u.slot : nullptr, lo_t ? lo_t + stride * u.slot : nullptr,
                                    bs->main);
                if (!lo && !hi_t) {
                }
            } else {
                launch_f64_to_f32(d, 1, rows, cols, base + stride * u.slot, R, Cc, bs->main);
            }
            CK(cudaStreamSynchronize(bs->main));
        };
        auto wr64 = [&](double* base, size_t stride, size_t cnt) {
            if (count < int64_t(cnt)) throw Fail{ASG_ERR_SHAPE_MISMATCH, "input too small"};
            if (!base) throw Fail{ASG_ERR_INVALID_ARGUMENT, "role not held by this method"};
            h2d(base + stride * u.slot, in, cnt * 8, bs->main);
        };
        const bool sp = split_mode(bs);
        switch (role) {
            case ASG_ROLE_FACTOR_L: wr32(g.L, slabMM(g), g.M, g.M, m, m, nullptr, nullptr, nullptr); break;
            case ASG_ROLE_FACTOR_R: wr32(g.R, slabNN(g), g.N, g.N, n, n, nullptr, nullptr, nullptr); break;
            case ASG_ROLE_INV_L:
                wr32(g.PLh, slabMM(g), g.M, g.M, m, m, sp ? g.PLl : nullptr, nullptr, nullptr);
                if (f16_mode(bs)) to_f16(g.PLh, g.nb, u.slot, 1, int64_t(slabMM(g)), g.PL16, g.plscale, g.amax2, bs->main,
                                          g.pln1, g.M);
                break;
            case ASG_ROLE_INV_R:
                wr32(g.PRh, slabNN(g), g.N, g.N, n, n, sp ? g.PRl : nullptr, nullptr, nullptr);
                if (f16_mode(bs)) to_f16(g.PRh, g.nb, u.slot, 1, int64_t(slabNN(g)), g.PR16, g.prscale, g.amax2, bs->main,
                                          g.prn1, g.N);
                break;
            case ASG_ROLE_KL_INV_L:
            case ASG_ROLE_KL_INV_R:
                throw Fail{ASG_ERR_INVALID_ARGUMENT,
                           "KL-Shampoo's F^-1 is derived from the installed root (INV^2); write ASG_ROLE_INV_*"};
            case ASG_ROLE_BASIS_L:
            case ASG_ROLE_BASIS_R: {
                const bool left = role == ASG_ROLE_BASIS_L;
                const int d = left ? m : n, D = left ? g.M : g.N;
                double* q64 = left ? g.QL64 : g.QR64;
                const double* src = nullptr;
                if (q64) {  // F64 refresh keeps the fp64 basis
                    wr64(q64, size_t(d) * d, size_t(d) * d);
                    src = q64 + size_t(d) * d * u.slot;
                } else {  // F32 refresh: split basis only; stage through the fp64 workspace
                    if (count < int64_t(d) * d) throw Fail{ASG_ERR_SHAPE_MISMATCH, "input too small"};
                    if (!g.QLh) throw Fail{ASG_ERR_INVALID_ARGUMENT, "role not held by this method"};
                    h2d(bs->ws_out, in, size_t(d) * d * 8, bs->main);
                    src = bs->ws_out;
                }
                const size_t DD = size_t(D) * D;
                launch_f64_to_split(src, 1, d, D, false, (left ? g.QLh : g.QRh) + DD * u.slot,
                                    sp ? (left ? g.QLl : g.QRl) + DD * u.slot : nullptr,
                                    (left ? g.QLTh : g.QRTh) + DD * u.slot,
                                    sp ? (left ? g.QLTl : g.QRTl) + DD * u.slot : nullptr, bs->main);
                break;
            }
            case ASG_ROLE_EIGVALS_L: wr64(g.valsL, size_t(m), size_t(m)); break;
            case ASG_ROLE_EIGVALS_R: wr64(g.valsR, size_t(n), size_t(n)); break;
            case ASG_ROLE_ROTATED_M: wr32(g.mom_m, slabMN(g), g.M, g.N, m, n, nullptr, nullptr, nullptr); break;
            case ASG_ROLE_ROTATED_V: wr32(g.mom_v, slabMN(g), g.M, g.N, m, n, nullptr, nullptr, nullptr); break;
            default: throw Fail{ASG_ERR_INVALID_ARGUMENT, "unknown role"};
        }
        CK(cudaStreamSynchronize(bs->main));
    });
}

int asg_block_set_counters(asg_blockset* bs, int64_t idx, uint64_t version, int64_t last_refresh_step, int64_t moment_steps) {
    return guard([&] {
        check_owned_index(bs, idx);
        Unit& u = bs->units[size_t(idx)];
        u.version = version;
        u.last_refresh_step = last_refresh_step;
        u.moment_steps = moment_steps;
    });
}

int asg_block_accumulate_f64(asg_blockset* bs, int64_t idx, const double* g, int64_t ld) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        check_owned_index(bs, idx);
        const Unit& u = bs->units[size_t(idx)];
        Group& gr = owned_group(bs, u);
        stage_host_grad(bs, u, g, ld);
        prep_single(bs, gr, u);
        group_stats(bs, gr, u.slot, 1, bs->main);
        CK(cudaStreamSynchronize(bs->main));
    });
}

int asg_block_refresh_f64(asg_blockset* bs, int64_t idx, int64_t step) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        check_owned_index(bs, idx);
        Unit& u = bs->units[size_t(idx)];
        owned_group(bs, u);
        if (u.pending) throw Fail{ASG_ERR_INVALID_ARGUMENT, "block has a pending scheduled refresh"};
        u.pending = true;
        u.launched = false;
        u.needs_launch = true;
        u.warm_start = u.version > 0;
        launch_refreshes(bs);
        try {
            install_device(bs, u);
        } catch (...) {
            u.pending = false;
            u.launched = false;
            u.needs_launch = false;
            throw;
        }
        u.pending = false;
        u.launched = false;
        u.version += 1;  // install_refresh precond.cpp:162-163
        u.last_refresh_step = step;
        CK(cudaStreamSynchronize(bs->main));
    });
}

int asg_block_precondition_f64(asg_blockset* bs, int64_t idx, const double* g, int64_t ld, double* out) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        check_owned_index(bs, idx);
        const Unit& u = bs->units[size_t(idx)];
        Group& gr = owned_group(bs, u);
        if (is_soap(bs)) throw Fail{ASG_ERR_INVALID_ARGUMENT, "use asg_block_soap_step_f64 for SOAP"};
        if (u.version == 0)  // precond.cpp:192-194
            throw Fail{ASG_ERR_STALE_UNINITIALIZED, "precondition_shampoo: no inverse installed"};
        stage_host_grad(bs, u, g, ld);
        prep_single(bs, gr, u);
        group_update(bs, gr, u.slot, 1, EPI_STORE, 0.f, nullptr, bs->d_out1, bs->main);
        download_block(bs, gr, out);
    });
}

int asg_block_soap_step_f64(asg_blockset* bs, int64_t idx, const double* g, int64_t ld, double* out) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        check_owned_index(bs, idx);
        Unit& u = bs->units[size_t(idx)];
        Group& gr = owned_group(bs, u);
        if (!is_soap(bs)) throw Fail{ASG_ERR_INVALID_ARGUMENT, "not a SOAP blockset"};
        stage_host_grad(bs, u, g, ld);
        prep_single(bs, gr, u);
        u.moment_steps += 1;  // precond.cpp:213
        group_update(bs, gr, u.slot, 1, EPI_STORE, 0.f, nullptr, bs->d_out1, bs->main);
        download_block(bs, gr, out);
    });
}

// ---- multi-GPU --------------------------------------------------------------
int asg_plan_owners(const asg_optimizer_config* opt, const int64_t* rows, const int64_t* cols, int64_t n_params,
                    int32_t world, int32_t* owner, int64_t capacity, int64_t* count) {
    return guard([&] {
        if (!opt || (n_params > 0 && (!rows || !cols)) || world < 1) throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad argument"};
        validate(*opt);
        asg_blockset tmp;  // host-side planning only: no device state is created
        tmp.opt = *opt;
        tmp.world = world;
        tmp.rank = 0;
        for (int64_t p = 0; p < n_params; ++p) {
            asg_param_desc d{};
            d.rows = rows[p];
            d.cols = cols[p];
            tmp.params.push_back(d);
        }
        build_units(&tmp);
        if (count) *count = int64_t(tmp.units.size());
        for (size_t i = 0; i < tmp.units.size() && int64_t(i) < capacity; ++i) owner[i] = tmp.units[i].owner;
    });
}

int asg_shard_elems(const asg_blockset* bs, int32_t rank, int64_t* elems) {
    return guard([&] {
        if (rank < 0 || rank >= bs->world) throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad rank"};
        *elems = bs->shard_elems[size_t(rank)];
    });
}

int asg_pack_owned(asg_blockset* bs, float* sendbuf, void* stream) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        launch_pack_blocks(bs->d_pack_refs, bs->d_pack_offs, bs->n_pack, sendbuf, s);
        CK(cudaGetLastError());
    });
}

int asg_unpack_gathered(asg_blockset* bs, const float* recvbuf, int64_t stride_elems, void* stream) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        if (stride_elems == bs->stride) {  // precomputed offsets (asg_gather_stride)
            launch_unpack_blocks(bs->d_unpack_refs, bs->d_unpack_offs, bs->n_unpack, recvbuf, s);
            CK(cudaGetLastError());
            return;
        }
        // offsets are within each rank's shard; ranks are `stride_elems` apart
        std::vector<int64_t> offs(size_t(bs->n_unpack));
        std::vector<int64_t> host_offs(size_t(bs->n_unpack));
        if (bs->n_unpack > 0)
            CK(cudaMemcpy(host_offs.data(), bs->d_unpack_offs, host_offs.size() * 8, cudaMemcpyDeviceToHost));
        for (int i = 0; i < bs->n_unpack; ++i)  // stored offsets use bs->stride: rebase
            offs[size_t(i)] = int64_t(bs->unpack_rank[size_t(i)]) * stride_elems +
                              (host_offs[size_t(i)] - int64_t(bs->unpack_rank[size_t(i)]) * bs->stride);
        int64_t* d_offs = nullptr;
        if (bs->n_unpack > 0) {
            CK(cudaMallocAsync(reinterpret_cast<void**>(&d_offs), offs.size() * 8, s));
            CK(cudaMemcpyAsync(d_offs, offs.data(), offs.size() * 8, cudaMemcpyHostToDevice, s));
            launch_unpack_blocks(bs->d_unpack_refs, d_offs, bs->n_unpack, recvbuf, s);
            CK(cudaFreeAsync(d_offs, s));
            CK(cudaStreamSynchronize(s));
        }
        CK(cudaGetLastError());
    });
}

int asg_gather_stride(const asg_blockset* bs, int64_t* stride) {
    return guard([&] {
        if (!bs || !stride) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        *stride = bs->stride;
    });
}

int asg_pack_grads(asg_blockset* bs, float* sendbuf, void* stream) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        if (bs->world > 1)  // padding between shards stays zero
            CK(cudaMemsetAsync(sendbuf, 0, size_t(bs->world) * bs->stride * 4, s));
        launch_pack_blocks(bs->d_gpack_refs, bs->d_gpack_offs, bs->n_unpack, sendbuf, s);
        CK(cudaGetLastError());
    });
}

int asg_unpack_reduced_grads(asg_blockset* bs, const float* recvbuf, float scale, void* stream) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        launch_unpack_scaled(bs->d_gunpack_refs, bs->d_gunpack_offs, bs->n_pack, recvbuf, scale, s);
        CK(cudaGetLastError());
    });
}

int asg_grad_sqnorm_owned(asg_blockset* bs, void* stream, double* sqnorm, int32_t* nonfinite) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        CK(cudaMemsetAsync(bs->d_sqnorm, 0, sizeof(double), s));
        CK(cudaMemsetAsync(bs->d_flag, 0, sizeof(int), s));
        for (const Unit& u : bs->units) {
            if (u.owner != bs->rank) continue;
            const asg_param_desc& d = bs->params[size_t(u.spec.param_index)];
            launch_sqnorm(d.grad + u.spec.row_begin * d.ld_grad + u.spec.col_begin, u.spec.row_end - u.spec.row_begin,
                          u.spec.col_end - u.spec.col_begin, d.ld_grad, bs->d_sqnorm, bs->d_flag, s);
        }
        double v = 0.0;
        int f = 0, fu = 0;
        CK(cudaMemcpyAsync(&v, bs->d_sqnorm, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&f, bs->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        // the previous step's update flag (s is ordered after the step that wrote it)
        CK(cudaMemcpyAsync(&fu, bs->d_upd_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaMemsetAsync(bs->d_flag, 0, sizeof(int), s));
        if (sqnorm) *sqnorm = v;
        if (nonfinite) *nonfinite = f;
        resolve_deferred(bs, false);
        if (fu) {
            CK(cudaMemsetAsync(bs->d_upd_flag, 0, sizeof(int), s));
            throw Fail{ASG_ERR_NON_FINITE, "apply_update: the previous step's update was non-finite "
                                           "(those elements of theta were left unchanged)"};
        }
    });
}

// ---- profiling ------------------------------------------------------------------
int asg_launch_count(uint64_t* count) {
    return guard([&] {
        if (!count) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        *count = launch_count();
    });
}

int asg_profile_enable(asg_blockset* bs, int32_t enable) {
    return guard([&] {
        bs->profiling = enable != 0;
        bs->launch_base = launch_count();
    });
}

int asg_get_hbm_stats(asg_blockset* bs, asg_hbm_stats* out, int32_t reset) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        CK(cudaStreamSynchronize(bs->main));
        sync_side(bs);
        CK(cudaDeviceSynchronize());  // the norm runs on the caller's stream
        *out = asg_hbm_stats{};
        for (auto& h : bs->prof_hbm) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, h.e0, h.e1));
            if (h.kind < 0 || h.kind >= ASG_HBM_KINDS) continue;
            out->launches[h.kind] += 1;
            out->bytes[h.kind] += h.bytes;
            out->ms[h.kind] += t;
        }
        if (reset) {
            for (auto& h : bs->prof_hbm) {
                cudaEventDestroy(h.e0);
                cudaEventDestroy(h.e1);
            }
            bs->prof_hbm.clear();
        }
    });
}

int asg_get_kernel_stats(asg_blockset* bs, asg_kernel_stats* out, int32_t reset) {
    return guard([&] {
        CK(cudaSetDevice(bs->device));
        CK(cudaStreamSynchronize(bs->main));
        sync_side(bs);
        double ms = 0.0;
        for (auto& e : bs->prof_events) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, e.first, e.second));
            ms += t;
        }
        out->launches = launch_count() - bs->launch_base;
        out->gemm_launches = bs->prof_gemms;
        out->gemm_alg_flops = bs->prof_flops;
        out->gemm_ms = ms;
        if (reset) {
            for (auto& e : bs->prof_events) {
                cudaEventDestroy(e.first);
                cudaEventDestroy(e.second);
            }
            bs->prof_events.clear();
            bs->prof_flops = 0.0;
            bs->prof_gemms = 0;
            bs->launch_base = launch_count();
        }
    });
}

// ---- diagnostics ------------------------------------------------------------
int asg_gemm_tn(const float* A, const float* B, float* C, int64_t batch, int64_t M, int64_t N, int64_t K, float alpha,
                float beta, int32_t precision, void* stream) {
    return guard([&] {
        if (M % 128 || N % 128 || K % 32 || batch < 1) throw Fail{ASG_ERR_SHAPE_MISMATCH, "M,N % 128 and K % 32 required"};
        int dev = 0;
        CK(cudaGetDevice(&dev));
        if (!asg_device_supported(dev)) throw Fail{ASG_ERR_UNSUPPORTED, "device is not sm_100"};
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, dev));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const bool sp = precision == ASG_PREC_3XTF32;
        // split operands into (hi, lo) slabs
        float *Ah = nullptr, *Al = nullptr, *Bh = nullptr, *Bl = nullptr;
        const size_t na = size_t(batch) * M * K, nbb = size_t(batch) * N * K;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&Ah), na * 4, s));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&Bh), nbb * 4, s));
        if (sp) {
            CK(cudaMallocAsync(reinterpret_cast<void**>(&Al), na * 4, s));
            CK(cudaMallocAsync(reinterpret_cast<void**>(&Bl), nbb * 4, s));
        }
        // reuse prep (identity scale, no transpose needed: write the transposes into scratch)
        float *scrA = nullptr, *scrB = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&scrA), na * 4 * (sp ? 2 : 1), s));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&scrB), nbb * 4 * (sp ? 2 : 1), s));
        std::vector<BlockRef> ra(static_cast<size_t>(batch)), rb(static_cast<size_t>(batch));
        for (int64_t b = 0; b < batch; ++b) {
            ra[size_t(b)] = BlockRef{A + b * M * K, nullptr, K, int32_t(M), int32_t(K)};
            rb[size_t(b)] = BlockRef{B + b * N * K, nullptr, K, int32_t(N), int32_t(K)};
        }
        BlockRef *dra = nullptr, *drb = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&dra), ra.size() * sizeof(BlockRef), s));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&drb), rb.size() * sizeof(BlockRef), s));
        CK(cudaMemcpyAsync(dra, ra.data(), ra.size() * sizeof(BlockRef), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(drb, rb.data(), rb.size() * sizeof(BlockRef), cudaMemcpyHostToDevice, s));
        launch_prep_grad(dra, int(batch), int(M), int(K), nullptr, 1.f, Ah, Al, scrA, sp ? scrA + na : nullptr, s);
        launch_prep_grad(drb, int(batch), int(N), int(K), nullptr, 1.f, Bh, Bl, scrB, sp ? scrB + nbb : nullptr, s);
        GemmLaunch g{};
        g.A = Operand{Ah, Al, int(M), int(K)};
        g.B = Operand{Bh, Bl, int(N), int(K)};
        float* scales = nullptr;
        unsigned int* amax = nullptr;
        if (precision == ASG_PREC_3XF16) {  // operands as fp16 pairs with per-matrix scales (in the scratch)
            CK(cudaMallocAsync(reinterpret_cast<void**>(&scales), size_t(batch) * 2 * sizeof(float), s));
            CK(cudaMallocAsync(reinterpret_cast<void**>(&amax), size_t(batch) * 2 * sizeof(unsigned int), s));
            launch_absmax(Ah, int(batch), M * K, amax, s);
            launch_absmax(Bh, int(batch), N * K, amax + batch, s);
            launch_to_f16pair(Ah, amax, int(batch), M * K, scrA, reinterpret_cast<uint16_t*>(scrA) + na, scales, s);
            launch_to_f16pair(Bh, amax + batch, int(batch), N * K, scrB, reinterpret_cast<uint16_t*>(scrB) + nbb,
                              scales + batch, s);
            g.A = Operand{scrA, reinterpret_cast<const float*>(reinterpret_cast<uint16_t*>(scrA) + na), int(M), int(K),
                          scales};
            g.B = Operand{scrB, reinterpret_cast<const float*>(reinterpret_cast<uint16_t*>(scrB) + nbb), int(N),
                          int(K), scales + batch};
        }
        g.batch = int(batch);
        g.epi = EPI_STORE;
        g.p.alpha = alpha;
        g.p.beta = beta;
        g.p.C = C;
        g.p.ldc = N;
        g.p.c_bstride = M * N;
        // diagnostics: ASG_GEMM_BENCH_REPS = k > 0 times the product, timed by CUDA events after one
        // warm-up launch; the mean kernel time goes to stderr (kernel-only, on prepared operands)
        static const int reps = getenv("ASG_GEMM_BENCH_REPS") ? std::max(0, atoi(getenv("ASG_GEMM_BENCH_REPS"))) : 0;
        CK(gemm_launch(g, precision, prop.multiProcessorCount, s));
        if (reps > 0) {
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0, s));
            for (int r = 0; r < reps; ++r) CK(gemm_launch(g, precision, prop.multiProcessorCount, s));
            CK(cudaEventRecord(e1, s));
            CK(cudaEventSynchronize(e1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            std::fprintf(stderr, "asg_gemm_tn bench: %d x (%lld x %lld x %lld x %lld) %.4f ms per launch\n", reps,
                         (long long)batch, (long long)M, (long long)N, (long long)K, ms / reps);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
        CK(cudaStreamSynchronize(s));
        for (void* p : {static_cast<void*>(Ah), static_cast<void*>(Al), static_cast<void*>(Bh), static_cast<void*>(Bl),
                        static_cast<void*>(scrA), static_cast<void*>(scrB), static_cast<void*>(dra), static_cast<void*>(drb),
                        static_cast<void*>(scales), static_cast<void*>(amax)})
            if (p) CK(cudaFreeAsync(p, s));
        CK(cudaStreamSynchronize(s));
    });
}

int asg_sym_eig_batched(const double* A, double* values, double* vectors, int64_t batch, int64_t n, void* stream) {
    return guard([&] {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        double* work = nullptr;
        int* status = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&work),
                           std::max(size_t(batch) * n * n, eigh_workspace_doubles(int(batch), int(n))) * 8, s));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&status), size_t(batch) * sizeof(int), s));
        CK(cudaMemsetAsync(status, 0, size_t(batch) * sizeof(int), s));
        launch_eigh(A, values, vectors, work, int(batch), int(n), status, s);
        std::vector<int> st(static_cast<size_t>(batch));
        CK(cudaMemcpyAsync(st.data(), status, st.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaFreeAsync(work, s));
        CK(cudaFreeAsync(status, s));
        CK(cudaStreamSynchronize(s));
        for (int v : st)
            if (v != ASG_OK) throw Fail{v, "sym_eig_batched: a matrix failed"};
    });
}

}  // extern "C"

namespace asg {
namespace {
// [b][n][n] <-> [b][D][D] (zero padding) for the fp32 diagnostic solve.
__global__ void pad_f32_kernel(const float* __restrict__ src, int n, int D, float* __restrict__ dst) {
    const int64_t b = blockIdx.y;
    const int64_t DD = int64_t(D) * D;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < DD; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e / D), j = int(e % D);
        dst[b * DD + e] = (i < n && j < n) ? src[b * int64_t(n) * n + int64_t(i) * n + j] : 0.f;
    }
}
__global__ void unpad_sum_kernel(const float* __restrict__ hi, const float* __restrict__ lo, int n, int D,
                                 float* __restrict__ dst) {
    const int64_t b = blockIdx.y;
    const int64_t nn = int64_t(n) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nn; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e / n), j = int(e % n);
        const int64_t o = b * int64_t(D) * D + int64_t(i) * D + j;
        dst[b * nn + e] = hi[o] + lo[o];
    }
}

// Scratch of the batched C-ABI solvers (asg_sym_eig_batched_f32 / asg_inv_root_batched_f32):
// one grow-only device buffer per device, held for the whole call (calls serialise on it), so
// a call neither maps fresh memory (a 100+ GB cudaMallocAsync per call dominated C5) nor
// re-captures the solvers' cached graphs (their keys hold the buffer pointers). Batches are
// processed in chunks that fit batched_scratch_bytes() (24 GiB).
size_t batched_scratch_bytes() {  // ASG_BATCHED_SCRATCH_BYTES: tests force small chunks
    static const size_t b = getenv("ASG_BATCHED_SCRATCH_BYTES") ? size_t(atoll(getenv("ASG_BATCHED_SCRATCH_BYTES")))
                                                               : (size_t(24) << 30);
    return b;
}
struct Arena {
    std::mutex mu;
    void* p = nullptr;
    size_t bytes = 0;
};
Arena& batched_arena(int dev) {
    static std::mutex m;
    static std::map<int, std::unique_ptr<Arena>> arenas;
    std::lock_guard<std::mutex> lk(m);
    auto& a = arenas[dev];
    if (!a) a = std::make_unique<Arena>();
    return *a;
}
// caller holds a.mu
char* arena_reserve(Arena& a, size_t bytes) {
    if (a.bytes < bytes) {
        if (a.p) {
            CK(cudaDeviceSynchronize());
            CK(cudaFree(a.p));
            a.p = nullptr;
            a.bytes = 0;
        }
        CK(cudaMalloc(&a.p, bytes));
        a.bytes = bytes;
    }
    return static_cast<char*>(a.p);
}
size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
}  // namespace
}  // namespace asg

int asg_sym_eig_batched_f32(const float* A, double* values, float* vectors, int64_t batch, int64_t n, void* stream) {
    return guard([&] {
        if (n <= kSmallEighN) throw Fail{ASG_ERR_UNSUPPORTED, "sym_eig_batched_f32: n must exceed 64"};
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        int dev = 0;
        CK(cudaGetDevice(&dev));
        int sms = 148;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int D = tc_eigh_dim(int(n));
        const size_t DD = size_t(D) * D;
        auto need = [&](int64_t c) {
            return align256(size_t(c) * DD * 4) + align256(4 * size_t(c) * DD * 4) +
                   align256(tc_eigh_workspace_floats(int(c), int(n)) * 4) + align256(size_t(c) * sizeof(int));
        };
        int64_t cb = batch;
        while (cb > 1 && need(cb) > batched_scratch_bytes()) cb = (cb + 1) / 2;
        Arena& ar = batched_arena(dev);
        std::lock_guard<std::mutex> lk(ar.mu);
        char* base = arena_reserve(ar, need(cb));
        std::vector<int> st(static_cast<size_t>(batch));
        for (int64_t b0 = 0; b0 < batch; b0 += cb) {
            const int64_t c = std::min(cb, batch - b0);
            const size_t nbDD = size_t(c) * DD;
            char* q = base;
            float* Bp = reinterpret_cast<float*>(q);
            q += align256(nbDD * 4);
            float* J = reinterpret_cast<float*>(q);
            q += align256(4 * nbDD * 4);
            float* ws = reinterpret_cast<float*>(q);
            q += align256(tc_eigh_workspace_floats(int(c), int(n)) * 4);
            int* status = reinterpret_cast<int*>(q);
            CK(cudaMemsetAsync(status, 0, size_t(c) * sizeof(int), s));
            pad_f32_kernel<<<dim3(256, unsigned(c)), 256, 0, s>>>(A + b0 * n * n, int(n), D, Bp);
            launch_tc_eigh(Bp, D, values + b0 * n, J, J + nbDD, J + 2 * nbDD, J + 3 * nbDD, ws, int(c), int(n), status,
                           sms, s, f32_refresh_tol());
            unpad_sum_kernel<<<dim3(256, unsigned(c)), 256, 0, s>>>(J, J + nbDD, int(n), D, vectors + b0 * n * n);
            count_launch(2);
            CK(cudaMemcpyAsync(st.data() + b0, status, size_t(c) * sizeof(int), cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        CK(cudaGetLastError());
        for (int v : st)
            if (v != ASG_OK) throw Fail{v, "sym_eig_batched_f32: a matrix failed"};
    });
}

int asg_inv_root_batched_f32(const float* A, float* out, int64_t batch, int64_t n, int32_t p, double damping,
                             int32_t precision, void* stream) {
    return guard([&] {
        if (n < 1 || batch < 1) throw Fail{ASG_ERR_INVALID_ARGUMENT, "inv_root_batched_f32: empty batch"};
        if (p != 2 && p != 4) throw Fail{ASG_ERR_INVALID_ARGUMENT, "inv_root_batched_f32: p must be 2 or 4"};
        if (n > 4096) throw Fail{ASG_ERR_UNSUPPORTED, "inv_root_batched_f32: n must be <= 4096"};
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        int dev = 0;
        CK(cudaGetDevice(&dev));
        int sms = 148;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int D = int(round_up(n, 128));
        const size_t DD = size_t(D) * D;
        const int bn = gemm_bn_for(D, int(std::min<int64_t>(batch, 1 << 20)));
        std::vector<int2> tl(size_t(gemm_sym_tile_list(D, bn, nullptr)));
        gemm_sym_tile_list(D, bn, tl.data());
        auto need = [&](int64_t c) {
            return align256(size_t(c) * DD * 4) + align256(2 * size_t(c) * DD * 4) +
                   align256(ns_workspace_floats(int(c), D) * 4) + align256(size_t(c) * 8) +
                   align256(size_t(c) * sizeof(int)) + align256(tl.size() * sizeof(int2));
        };
        int64_t cb = batch;
        while (cb > 1 && need(cb) > batched_scratch_bytes()) cb = (cb + 1) / 2;
        Arena& ar = batched_arena(dev);
        std::lock_guard<std::mutex> lk(ar.mu);
        char* base = arena_reserve(ar, need(cb));
        std::vector<int> st(static_cast<size_t>(batch));
        for (int64_t b0 = 0; b0 < batch; b0 += cb) {
            const int64_t c = std::min(cb, batch - b0);
            const size_t nbDD = size_t(c) * DD;
            char* q = base;
            auto take = [&](size_t b) {
                char* r = q;
                q += align256(b);
                return r;
            };
            float* Ap = reinterpret_cast<float*>(take(nbDD * 4));
            float* R = reinterpret_cast<float*>(take(2 * nbDD * 4));
            float* ws = reinterpret_cast<float*>(take(ns_workspace_floats(int(c), D) * 4));
            double* eps = reinterpret_cast<double*>(take(size_t(c) * 8));
            int* status = reinterpret_cast<int*>(take(size_t(c) * sizeof(int)));
            int2* tiles = reinterpret_cast<int2*>(take(tl.size() * sizeof(int2)));
            CK(cudaMemcpyAsync(tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
            CK(cudaMemsetAsync(status, 0, size_t(c) * sizeof(int), s));
            pad_f32_kernel<<<dim3(256, unsigned(c)), 256, 0, s>>>(A + b0 * n * n, int(n), D, Ap);
            count_launch(1);
            launch_relative_damping_f32(Ap, int(c), D, int(n), damping, eps, s);
            launch_ns_inv_root(Ap, int(c), int(n), D, eps, p, R, precision == ASG_PREC_3XTF32 ? R + nbDD : nullptr, ws,
                               status, tiles, int(tl.size()), precision, sms, s);
            if (precision != ASG_PREC_3XTF32) CK(cudaMemsetAsync(R + nbDD, 0, nbDD * 4, s));
            unpad_sum_kernel<<<dim3(256, unsigned(c)), 256, 0, s>>>(R, R + nbDD, int(n), D, out + b0 * n * n);
            count_launch(1);
            CK(cudaMemcpyAsync(st.data() + b0, status, size_t(c) * sizeof(int), cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        CK(cudaGetLastError());
        for (int v : st)
            if (v != ASG_OK) throw Fail{v, "inv_root_batched_f32: a matrix failed"};
    });
}

// ---- NCCL and the bucketed parameter all-gather -------
int asg_nccl_unique_id(uint8_t* out) {
    return guard([&] {
        if (!out) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null output"};
        ncclUniqueId id;
        nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int asg_nccl_comm_init(int32_t world, int32_t rank, const uint8_t* id, void** comm) {
    return guard([&] {
        if (!id || !comm || world < 1 || rank < 0 || rank >= world) throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad arguments"};
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
        ncclComm_t c = nullptr;
        nccl_check(nccl().CommInitRank(&c, world, uid, rank), "ncclCommInitRank");
        *comm = c;
    });
}

int asg_nccl_comm_destroy(void* comm) {
    return guard([&] {
        if (comm) nccl_check(nccl().CommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
    });
}

int asg_set_allgather_buckets(asg_blockset* bs, int32_t buckets_per_shape) {
    return guard([&] {
        if (!bs || buckets_per_shape < 1) throw Fail{ASG_ERR_INVALID_ARGUMENT, "buckets_per_shape must be >= 1"};
        CK(cudaSetDevice(bs->device));
        CK(cudaStreamSynchronize(bs->main));
        build_buckets(bs, buckets_per_shape);
        for (cudaEvent_t e : bs->ag_events) cudaEventDestroy(e);
        bs->ag_events.assign(bs->buckets.size(), nullptr);
        for (cudaEvent_t& e : bs->ag_events) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    });
}

int asg_bucket_count(const asg_blockset* bs, int64_t* count) {
    return guard([&] {
        if (!bs || !count) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        *count = int64_t(bs->buckets.size());
    });
}

int asg_bucket_stride(const asg_blockset* bs, int64_t bucket, int64_t* stride) {
    return guard([&] {
        if (!bs || !stride || bucket < 0 || bucket >= int64_t(bs->buckets.size()))
            throw Fail{ASG_ERR_INVALID_ARGUMENT, "bucket index out of range"};
        *stride = bs->buckets[size_t(bucket)].stride;
    });
}

int asg_bucket_pack(asg_blockset* bs, int64_t bucket, float* sendbuf, void* stream) {
    return guard([&] {
        if (!bs || bucket < 0 || bucket >= int64_t(bs->buckets.size()))
            throw Fail{ASG_ERR_INVALID_ARGUMENT, "bucket index out of range"};
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        const auto& b = bs->buckets[size_t(bucket)];
        launch_pack_blocks(b.d_pack_refs, b.d_pack_offs, b.n_pack, sendbuf, s);
        CK(cudaGetLastError());
    });
}

int asg_bucket_unpack(asg_blockset* bs, int64_t bucket, const float* recvbuf, void* stream) {
    return guard([&] {
        if (!bs || bucket < 0 || bucket >= int64_t(bs->buckets.size()))
            throw Fail{ASG_ERR_INVALID_ARGUMENT, "bucket index out of range"};
        CK(cudaSetDevice(bs->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        const auto& b = bs->buckets[size_t(bucket)];
        launch_unpack_blocks(b.d_unpack_refs, b.d_unpack_offs, b.n_unpack, recvbuf, s);
        CK(cudaGetLastError());
    });
}

int asg_set_allgather_comm(asg_blockset* bs, void* comm, int32_t buckets_per_shape) {
    return guard([&] {
        if (!bs) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null blockset"};
        CK(cudaSetDevice(bs->device));
        if (comm) {
            nccl();  // fail now if NCCL cannot be loaded
            if (buckets_per_shape < 1) throw Fail{ASG_ERR_INVALID_ARGUMENT, "buckets_per_shape must be >= 1"};
            if (int(bs->buckets.size()) == 0 || bs->buckets_per_shape != buckets_per_shape) {
                if (int rc = asg_set_allgather_buckets(bs, buckets_per_shape)) throw Fail{rc, g_err};
            }
            if (!bs->comm_stream) {
                int lo = 0, hi = 0;
                CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
                CK(cudaStreamCreateWithPriority(&bs->comm_stream, cudaStreamNonBlocking, hi));
                CK(cudaEventCreateWithFlags(&bs->ag_done, cudaEventDisableTiming));
            }
        }
        bs->ag_comm = comm;
    });
}

int asg_allgather_params(asg_blockset* bs, void* comm, void* stream) {
    return guard([&] {
        if (!bs || !comm) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null blockset or communicator"};
        CK(cudaSetDevice(bs->device));
        if (bs->buckets.empty()) {
            if (int rc = asg_set_allgather_buckets(bs, 1)) throw Fail{rc, g_err};
        }
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : bs->main;
        if (s != bs->main) {  // after the step's update
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CK(cudaEventRecord(e, bs->main));
            CK(cudaStreamWaitEvent(s, e, 0));
            CK(cudaEventDestroy(e));
        }
        for (const auto& b : bs->buckets) bucket_exchange(bs, b, static_cast<ncclComm_t>(comm), s);
        CK(cudaGetLastError());
    });
}

// ---- split refresh API: snapshot_factors / compute_refresh / install_refresh
// (precond.hpp:90-98, precond.cpp:112-164) ------------------------------------
struct asg_snapshot {
    int64_t idx = 0;
    int M = 0, N = 0, m = 0, n = 0;
    float *L = nullptr, *R = nullptr;  // device copies of the padded factor slabs
};

struct asg_refresh_result {
    int64_t idx = 0;
    int method = 0;
    bool f64_soap = false;
    std::vector<void*> bufs;  // device
    // roots (Shampoo / KL-Shampoo): P per side, split pairs (KL: F^-1 = P^2)
    float *PLh = nullptr, *PLl = nullptr, *PRh = nullptr, *PRl = nullptr;
    // SOAP, F32 refresh: the new bases transposed (split); F64 refresh: the new bases (fp64)
    float *QLTh = nullptr, *QLTl = nullptr, *QRTh = nullptr, *QRTl = nullptr;
    double *QL64 = nullptr, *QR64 = nullptr, *valsL = nullptr, *valsR = nullptr;
};

namespace {
template <class T>
T* ralloc(asg_refresh_result* r, size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
    r->bufs.push_back(p);
    return static_cast<T*>(p);
}
void free_result(asg_refresh_result* r) {
    if (!r) return;
    for (void* p : r->bufs) cudaFree(p);
    delete r;
}
void d2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (dst && src && bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
}
uint64_t fnv1a64(const void* data, size_t n, uint64_t h = 0xcbf29ce484222325ull) {  // bytes.hpp:14-22
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}
}  // namespace

int asg_snapshot_factors(asg_blockset* bs, int64_t idx, asg_snapshot** out) {
    return guard([&] {
        if (!bs || !out) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        CK(cudaSetDevice(bs->device));
        check_owned_index(bs, idx);
        const Unit& u = bs->units[size_t(idx)];
        Group& g = owned_group(bs, u);
        auto* sn = new asg_snapshot();
        sn->idx = idx;
        sn->M = g.M;
        sn->N = g.N;
        sn->m = g.m;
        sn->n = g.n;
        cudaError_t e1 = cudaMalloc(reinterpret_cast<void**>(&sn->L), slabMM(g) * 4);
        cudaError_t e2 = cudaMalloc(reinterpret_cast<void**>(&sn->R), slabNN(g) * 4);
        if (e1 != cudaSuccess || e2 != cudaSuccess) {
            cudaFree(sn->L);
            cudaFree(sn->R);
            delete sn;
            throw Fail{ASG_ERR_OUT_OF_MEMORY, "snapshot_factors: device allocation failed"};
        }
        d2d(sn->L, at(g.L, slabMM(g), u.slot), slabMM(g) * 4, bs->main);
        d2d(sn->R, at(g.R, slabNN(g), u.slot), slabNN(g) * 4, bs->main);
        CK(cudaStreamSynchronize(bs->main));
        *out = sn;
    });
}

int asg_snapshot_checksum(const asg_snapshot* sn, uint64_t* out) {
    return guard([&] {
        if (!sn || !out) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        auto side = [&](const float* d, int D, int k) {
            std::vector<float> h(size_t(D) * D);
            CK(cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost));
            uint64_t x = 0xcbf29ce484222325ull;
            for (int i = 0; i < k; ++i) x = fnv1a64(h.data() + size_t(i) * D, size_t(k) * 4, x);
            return x;
        };
        const uint64_t hl = side(sn->L, sn->M, sn->m), hr = side(sn->R, sn->N, sn->n);
        *out = hr ^ (hl * 0x9e3779b97f4a7c15ull);  // snapshot_checksum precond.cpp:114-115
    });
}

int asg_snapshot_destroy(asg_snapshot* sn) {
    if (!sn) return ASG_OK;
    cudaFree(sn->L);
    cudaFree(sn->R);
    delete sn;
    return ASG_OK;
}

int asg_compute_refresh(asg_blockset* bs, const asg_snapshot* sn, asg_refresh_result** out) {
    asg_refresh_result* r = nullptr;
    const int rc = guard([&] {
        if (!bs || !sn || !out) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        CK(cudaSetDevice(bs->device));
        check_owned_index(bs, sn->idx);
        Unit& u = bs->units[size_t(sn->idx)];
        Group& g = owned_group(bs, u);
        if (g.M != sn->M || g.N != sn->N) throw Fail{ASG_ERR_SHAPE_MISMATCH, "compute_refresh: snapshot shape"};
        if (u.pending || u.needs_launch || u.launched)
            throw Fail{ASG_ERR_INVALID_ARGUMENT, "compute_refresh: block has a scheduled refresh in flight"};
        CK(cudaStreamSynchronize(bs->main));
        sync_side(bs);
        const size_t mm = slabMM(g), nn = slabNN(g);
        d2d(at(g.snapL, mm, u.slot), sn->L, mm * 4, bs->main);
        d2d(at(g.snapR, nn, u.slot), sn->R, nn * 4, bs->main);
        u.snap_preloaded = true;
        u.needs_launch = true;
        u.warm_start = u.version > 0;
        launch_refreshes(bs);
        CK(cudaEventSynchronize(u.done));
        u.launched = false;
        const int st = g.h_status[u.slot];
        if (st != ASG_OK) throw Fail{st, "compute_refresh: refresh failed"};
        r = new asg_refresh_result();
        r->idx = sn->idx;
        r->method = bs->opt.method;
        cudaStream_t s = bs->side;
        const bool sp = split_mode(bs);
        if (!is_soap(bs)) {
            r->PLh = ralloc<float>(r, mm);
            r->PRh = ralloc<float>(r, nn);
            d2d(r->PLh, at(g.sPLh, mm, u.slot), mm * 4, s);
            d2d(r->PRh, at(g.sPRh, nn, u.slot), nn * 4, s);
            if (sp) {
                r->PLl = ralloc<float>(r, mm);
                r->PRl = ralloc<float>(r, nn);
                d2d(r->PLl, at(g.sPLl, mm, u.slot), mm * 4, s);
                d2d(r->PRl, at(g.sPRl, nn, u.slot), nn * 4, s);
            }
        } else if (f32_refresh(bs)) {
            // absolute new bases, transposed: Q_new^T = J^T Q_cur^T (A = J^T, B = Q_cur)
            r->valsL = ralloc<double>(r, size_t(g.m));
            r->valsR = ralloc<double>(r, size_t(g.n));
            d2d(r->valsL, at(g.svalsL, size_t(g.m), u.slot), size_t(g.m) * 8, s);
            d2d(r->valsR, at(g.svalsR, size_t(g.n), u.slot), size_t(g.n) * 8, s);
            for (int side = 0; side < 2; ++side) {
                const bool left = side == 0;
                const int D = left ? g.M : g.N, d = left ? g.m : g.n;
                const size_t DD = size_t(D) * D;
                float* th = ralloc<float>(r, DD);
                float* tl = sp ? ralloc<float>(r, DD) : nullptr;
                (left ? r->QLTh : r->QRTh) = th;
                (left ? r->QLTl : r->QRTl) = tl;
                GemmParams p{};
                p.alpha = 1.f;
                p.Dhi = th;
                p.Dlo = tl;
                p.ldd = D;
                p.d_bstride = int64_t(DD);
                run_gemm(bs, op(at(left ? g.sJLTh : g.sJRTh, DD, u.slot), at(left ? g.sJLTl : g.sJRTl, DD, u.slot), D, D),
                         op(at(left ? g.QLh : g.QRh, DD, u.slot), at(left ? g.QLl : g.QRl, DD, u.slot), D, D), 1,
                         EPI_SPLIT, p, nullptr, 0, s, 2.0 * double(d) * d * d);
            }
        } else {
            r->f64_soap = true;
            const size_t dm = size_t(g.m) * g.m, dn = size_t(g.n) * g.n;
            r->QL64 = ralloc<double>(r, dm);
            r->QR64 = ralloc<double>(r, dn);
            r->valsL = ralloc<double>(r, size_t(g.m));
            r->valsR = ralloc<double>(r, size_t(g.n));
            d2d(r->QL64, at(g.sQL64, dm, u.slot), dm * 8, s);
            d2d(r->QR64, at(g.sQR64, dn, u.slot), dn * 8, s);
            d2d(r->valsL, at(g.svalsL, size_t(g.m), u.slot), size_t(g.m) * 8, s);
            d2d(r->valsR, at(g.svalsR, size_t(g.n), u.slot), size_t(g.n) * 8, s);
        }
        CK(cudaStreamSynchronize(s));
        *out = r;
        r = nullptr;
    });
    free_result(r);
    return rc;
}

int asg_install_refresh(asg_blockset* bs, int64_t idx, asg_refresh_result* r, int64_t step) {
    return guard([&] {
        if (!bs || !r) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        CK(cudaSetDevice(bs->device));
        check_owned_index(bs, idx);
        Unit& u = bs->units[size_t(idx)];
        Group& g = owned_group(bs, u);
        if (r->idx != idx || r->method != bs->opt.method)
            throw Fail{ASG_ERR_SHAPE_MISMATCH, "install_refresh: result of another block or method"};
        if (u.pending || u.launched) throw Fail{ASG_ERR_INVALID_ARGUMENT, "install_refresh: a scheduled refresh is in flight"};
        sync_side(bs);
        cudaStream_t s = bs->main;
        const size_t mm = slabMM(g), nn = slabNN(g);
        u.version += 1;  // install_refresh precond.cpp:162-163 (SOAP installs read the bumped version)
        u.last_refresh_step = step;
        if (!is_soap(bs)) {
            d2d(at(g.sPLh, mm, u.slot), r->PLh, mm * 4, s);
            d2d(at(g.sPRh, nn, u.slot), r->PRh, nn * 4, s);
            d2d(at(g.sPLl, mm, u.slot), r->PLl, mm * 4, s);
            d2d(at(g.sPRl, nn, u.slot), r->PRl, nn * 4, s);
            install_roots(bs, g, u.slot, 1);
        } else if (!r->f64_soap) {
            // rot = Q_new^T Q_old (precond.cpp:146-147) as the shadow rotation J^T:
            // A = Q_new^T (result), B = Q_old^T (the block's transposed basis)
            for (int side = 0; side < 2; ++side) {
                const bool left = side == 0;
                const int D = left ? g.M : g.N, d = left ? g.m : g.n;
                const size_t DD = size_t(D) * D;
                GemmParams p{};
                p.alpha = 1.f;
                p.Dhi = at(left ? g.sJLTh : g.sJRTh, DD, u.slot);
                p.Dlo = at(left ? g.sJLTl : g.sJRTl, DD, u.slot);
                p.ldd = D;
                p.d_bstride = int64_t(DD);
                run_gemm(bs, op(left ? r->QLTh : r->QRTh, left ? r->QLTl : r->QRTl, D, D),
                         op(at(left ? g.QLTh : g.QRTh, DD, u.slot), at(left ? g.QLTl : g.QRTl, DD, u.slot), D, D), 1,
                         EPI_SPLIT, p, nullptr, 0, s, 2.0 * double(d) * d * d);
            }
            d2d(at(g.svalsL, size_t(g.m), u.slot), r->valsL, size_t(g.m) * 8, s);
            d2d(at(g.svalsR, size_t(g.n), u.slot), r->valsR, size_t(g.n) * 8, s);
            install_soap_f32(bs, g, u.slot, 1);
        } else {
            const size_t dm = size_t(g.m) * g.m, dn = size_t(g.n) * g.n;
            d2d(at(g.sQL64, dm, u.slot), r->QL64, dm * 8, s);
            d2d(at(g.sQR64, dn, u.slot), r->QR64, dn * 8, s);
            d2d(at(g.svalsL, size_t(g.m), u.slot), r->valsL, size_t(g.m) * 8, s);
            d2d(at(g.svalsR, size_t(g.n), u.slot), r->valsR, size_t(g.n) * 8, s);
            install_apply(bs, u);
        }
        CK(cudaStreamSynchronize(s));
        free_result(r);  // consumed (RefreshResult&&)
    });
}

int asg_refresh_result_destroy(asg_refresh_result* r) {
    free_result(r);
    return ASG_OK;
}

// ---- replicated_state / load_replicated_state (precond.cpp:253-279) --------
int asg_block_replicated_state(asg_blockset* bs, int64_t idx, double* out, int64_t count) {
    return guard([&] {
        if (!bs || !out) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        check_owned_index(bs, idx);
        const Unit& u = bs->units[size_t(idx)];
        owned_group(bs, u);
        const int64_t nr = u.spec.row_end - u.spec.row_begin, nc = u.spec.col_end - u.spec.col_begin;
        if (count < nr * nr + nc * nc) throw Fail{ASG_ERR_SHAPE_MISMATCH, "replicated_state: output too small"};
        const bool soap = is_soap(bs);
        if (int rc = asg_block_read(bs, idx, soap ? ASG_ROLE_BASIS_L : ASG_ROLE_INV_L, out, nr * nr)) throw Fail{rc, g_err};
        if (int rc = asg_block_read(bs, idx, soap ? ASG_ROLE_BASIS_R : ASG_ROLE_INV_R, out + nr * nr, nc * nc))
            throw Fail{rc, g_err};
    });
}

int asg_block_load_replicated_state(asg_blockset* bs, int64_t idx, const double* in, int64_t count) {
    return guard([&] {
        if (!bs || !in) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        check_owned_index(bs, idx);
        const Unit& u = bs->units[size_t(idx)];
        owned_group(bs, u);
        const int64_t nr = u.spec.row_end - u.spec.row_begin, nc = u.spec.col_end - u.spec.col_begin;
        if (count != nr * nr + nc * nc) throw Fail{ASG_ERR_SHAPE_MISMATCH, "load_replicated_state: size mismatch"};
        const bool soap = is_soap(bs);
        if (int rc = asg_block_write(bs, idx, soap ? ASG_ROLE_BASIS_L : ASG_ROLE_INV_L, in, nr * nr)) throw Fail{rc, g_err};
        if (int rc = asg_block_write(bs, idx, soap ? ASG_ROLE_BASIS_R : ASG_ROLE_INV_R, in + nr * nr, nc * nc))
            throw Fail{rc, g_err};
    });
}

// ---- packed symmetric storage (pack_spd / unpack_spd densela.hpp:124-142) ----
namespace asg {
namespace {
// packed lower triangle, row-major: (0,0), (1,0), (1,1), (2,0), ...
__global__ void pack_spd_kernel(const float* __restrict__ A, int n, float* __restrict__ P) {
    const int i = blockIdx.x;
    const int64_t b = blockIdx.y;
    const float* row = A + (b * n + i) * int64_t(n);
    float* dst = P + b * (int64_t(n) * (n + 1) / 2) + int64_t(i) * (i + 1) / 2;
    for (int j = threadIdx.x; j <= i; j += blockDim.x) dst[j] = row[j];
}
__global__ void unpack_spd_kernel(const float* __restrict__ P, int n, float* __restrict__ A) {
    const int i = blockIdx.x;
    const int64_t b = blockIdx.y;
    const float* pk = P + b * (int64_t(n) * (n + 1) / 2);
    float* row = A + (b * n + i) * int64_t(n);
    for (int j = threadIdx.x; j < n; j += blockDim.x)
        row[j] = j <= i ? pk[int64_t(i) * (i + 1) / 2 + j] : pk[int64_t(j) * (j + 1) / 2 + i];
}
}  // namespace
}  // namespace asg

int asg_pack_spd_f32(const float* A, int64_t batch, int64_t n, float* packed, void* stream) {
    return guard([&] {
        if (!A || !packed || n < 1 || batch < 1 || n > 65535) throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad arguments"};
        pack_spd_kernel<<<dim3(unsigned(n), unsigned(batch)), 256, 0, static_cast<cudaStream_t>(stream)>>>(A, int(n),
                                                                                                        packed);
        count_launch();
        CK(cudaGetLastError());
    });
}

int asg_unpack_spd_f32(const float* packed, int64_t batch, int64_t n, float* A, void* stream) {
    return guard([&] {
        if (!A || !packed || n < 1 || batch < 1 || n > 65535) throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad arguments"};
        unpack_spd_kernel<<<dim3(unsigned(n), unsigned(batch)), 256, 0, static_cast<cudaStream_t>(stream)>>>(packed,
                                                                                                          int(n), A);
        count_launch();
        CK(cudaGetLastError());
    });
}

// ---- adamw_step / apply_update with host matrices (precond.cpp:229-251) ----
struct asg_adam_state {
    int64_t rows = 0, cols = 0, t = 0;
    float *m = nullptr, *v = nullptr;
};

namespace asg {
namespace {
__global__ void adamw_dir_kernel(const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v, int64_t n,
                                 float b1, float b2, float inv_bc1, float inv_bc2, float eps, float* __restrict__ out) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const float mm = b1 * m[e] + (1.f - b1) * g[e];
        const float vv = b2 * v[e] + (1.f - b2) * g[e] * g[e];
        m[e] = mm;
        v[e] = vv;
        out[e] = (mm * inv_bc1) / (sqrtf(vv * inv_bc2) + eps);
    }
}
__global__ void apply_update_kernel(double* __restrict__ theta, const double* __restrict__ u, int64_t n, double lr,
                                    double wd) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
        theta[e] -= lr * (u[e] + wd * theta[e]);
}
}  // namespace
}  // namespace asg

int asg_adam_state_create(int64_t rows, int64_t cols, asg_adam_state** out) {
    return guard([&] {
        if (!out || rows < 1 || cols < 1) throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad arguments"};
        auto* st = new asg_adam_state();
        st->rows = rows;
        st->cols = cols;
        const size_t n = size_t(rows * cols);
        if (cudaMalloc(reinterpret_cast<void**>(&st->m), n * 4) != cudaSuccess ||
            cudaMalloc(reinterpret_cast<void**>(&st->v), n * 4) != cudaSuccess) {
            cudaFree(st->m);
            cudaFree(st->v);
            delete st;
            throw Fail{ASG_ERR_OUT_OF_MEMORY, "adam state allocation failed"};
        }
        CK(cudaMemset(st->m, 0, n * 4));
        CK(cudaMemset(st->v, 0, n * 4));
        *out = st;
    });
}

int asg_adam_state_destroy(asg_adam_state* st) {
    if (!st) return ASG_OK;
    cudaFree(st->m);
    cudaFree(st->v);
    delete st;
    return ASG_OK;
}

int asg_adamw_step_f64(asg_adam_state* st, const double* g, const asg_optimizer_config* cfg, double* out) {
    return guard([&] {
        if (!st || !g || !cfg || !out) throw Fail{ASG_ERR_INVALID_ARGUMENT, "null argument"};
        const size_t n = size_t(st->rows * st->cols);
        std::vector<float> gf(n);
        for (size_t i = 0; i < n; ++i) {
            if (!std::isfinite(g[i])) throw Fail{ASG_ERR_NON_FINITE, "adamw_step: non-finite gradient"};
            gf[i] = float(g[i]);
        }
        float *dg = nullptr, *dout = nullptr;
        CK(cudaMalloc(reinterpret_cast<void**>(&dg), n * 4));
        CK(cudaMalloc(reinterpret_cast<void**>(&dout), n * 4));
        CK(cudaMemcpy(dg, gf.data(), n * 4, cudaMemcpyHostToDevice));
        st->t += 1;
        const double t = double(st->t);
        adamw_dir_kernel<<<256, 256>>>(dg, st->m, st->v, int64_t(n), float(cfg->beta1), float(cfg->beta2),
                                       float(1.0 / (1.0 - std::pow(cfg->beta1, t))),
                                       float(1.0 / (1.0 - std::pow(cfg->beta2, t))), float(cfg->eps), dout);
        count_launch();
        CK(cudaMemcpy(gf.data(), dout, n * 4, cudaMemcpyDeviceToHost));
        cudaFree(dg);
        cudaFree(dout);
        for (size_t i = 0; i < n; ++i) out[i] = double(gf[i]);
    });
}

int asg_apply_update_f64(double* theta, const double* update, int64_t rows, int64_t cols,
                         const asg_optimizer_config* cfg, double lr_scale) {
    return guard([&] {
        if (!theta || !update || !cfg || rows < 0 || cols < 0) throw Fail{ASG_ERR_INVALID_ARGUMENT, "bad arguments"};
        const size_t n = size_t(rows * cols);
        for (size_t i = 0; i < n; ++i)
            if (!std::isfinite(update[i])) throw Fail{ASG_ERR_NON_FINITE, "apply_update: non-finite update"};
        if (n == 0) return;
        double *dt = nullptr, *du = nullptr;
        CK(cudaMalloc(reinterpret_cast<void**>(&dt), n * 8));
        CK(cudaMalloc(reinterpret_cast<void**>(&du), n * 8));
        CK(cudaMemcpy(dt, theta, n * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(du, update, n * 8, cudaMemcpyHostToDevice));
        apply_update_kernel<<<256, 256>>>(dt, du, int64_t(n), cfg->lr * lr_scale, cfg->weight_decay);
        count_launch();
        CK(cudaMemcpy(theta, dt, n * 8, cudaMemcpyDeviceToHost));
        cudaFree(dt);
        cudaFree(du);
    });
}
