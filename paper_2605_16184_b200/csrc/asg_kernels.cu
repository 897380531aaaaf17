// SPDX-License-Identifier: Apache-2.0
//
// Device kernels of the optimizer step (all sm_100a) and their launchers.
//
//   GEMM          tcgen05 3xTF32/TF32 batched TN GEMM (asg_gemm.cuh), fused epilogues
//   K1 prep       gradient gather + clip scale + tf32 (hi, lo) split + transpose
//   K8 snapshot   factor slab -> fp64 shadow (snapshot_factors precond.cpp:112-117)
//   K6 eigh       batched symmetric eigendecomposition, fp64 (sym_eig densela.hpp:182-264)
//   K6 roots      (lam + eps)^p reconstruction (inv_root densela.hpp:267-282)
//   K9 adamw      AdamW + apply for 1-D parameters (precond.cpp:229-251)
//   K10 sqnorm    global gradient norm + non-finite flag (harness.cpp:219-223)
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "../../include/asteria_b200.h"
#include "asg_kernels.cuh"

namespace asg {

namespace {
std::atomic<uint64_t> g_launches{0};
}
uint64_t launch_count() { return g_launches.load(); }
void count_launch(uint64_t n) { g_launches.fetch_add(n); }

// ============================================================================
// GEMM launcher
// ============================================================================
namespace {

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled encode_fn() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    return fn;
}

// 3-D map over a [batch][rows][K] fp32 slab with a (32 x box_rows x 1) box,
// 128-byte swizzle (matches the UMMA K-major SWIZZLE_128B descriptor).
bool make_map(CUtensorMap* map, const float* base, int K, int rows, int batch, int box_rows, bool f16 = false) {
    PFN_encodeTiled enc = encode_fn();
    if (!enc) return false;
    const cuuint64_t es = f16 ? 2 : 4;  // element bytes; a box row is 128 bytes either way
    cuuint64_t dims[3] = {cuuint64_t(K), cuuint64_t(rows), cuuint64_t(batch)};
    cuuint64_t strides[2] = {cuuint64_t(K) * es, cuuint64_t(K) * cuuint64_t(rows) * es};
    cuuint32_t box[3] = {cuuint32_t(128 / es), cuuint32_t(box_rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                     const_cast<float*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int BN, int NPASS, int EPI, int CG, bool SPL, bool F16>
cudaError_t launch_inst(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                        const CUtensorMap& bl, const GemmParams& p, int num_sms, cudaStream_t s) {
    using Cfg = GemmCfg<BN, NPASS, CG, SPL, F16>;
    auto kern = gemm_tn_kernel<BN, NPASS, EPI, CG, SPL, F16>;
    // the shared-memory limit is a per-device function attribute; so is the
    // number of CTA pairs that can be co-resident (GPCs with an odd SM count)
    static std::atomic<uint64_t> attr_set{0};
    static int max_pairs[64] = {};
    int dev = 0;
    cudaError_t de = cudaGetDevice(&dev);
    if (de != cudaSuccess) return de;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (!(attr_set.load() & bit)) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::kSmemBytes));
        if (e != cudaSuccess) return e;
        if (CG == 2) {
            cudaLaunchConfig_t qc = {};
            qc.gridDim = dim3(2 * 74, 1, 1);
            qc.blockDim = dim3(Cfg::kThreads, 1, 1);
            qc.dynamicSmemBytes = Cfg::kSmemBytes;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = 2;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            qc.attrs = qa;
            qc.numAttrs = 1;
            int n = 0;
            e = cudaOccupancyMaxActiveClusters(&n, kern, &qc);
            if (e != cudaSuccess) return e;
            max_pairs[dev & 63] = n;
        }
        attr_set.fetch_or(bit);
    }
    if (p.num_tiles <= 0) return cudaSuccess;
    if (CG == 1) {
        const int grid = p.num_tiles < num_sms ? p.num_tiles : num_sms;
        kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, s>>>(ah, al, bh, bl, p);
    } else {
        int pairs = max_pairs[dev & 63];
        if (pairs > num_sms / 2) pairs = num_sms / 2;
        static const int cap = getenv("ASG_GEMM_MAX_PAIRS") ? atoi(getenv("ASG_GEMM_MAX_PAIRS")) : 0;  // tuning
        if (cap > 0 && pairs > cap) pairs = cap;
        if (pairs > p.num_tiles) pairs = p.num_tiles;
        if (pairs <= 0) return cudaErrorInvalidConfiguration;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * pairs, 1, 1);
        cfg.blockDim = dim3(Cfg::kThreads, 1, 1);
        cfg.dynamicSmemBytes = Cfg::kSmemBytes;
        cfg.stream = s;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 2;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ah, al, bh, bl, p);
        if (e != cudaSuccess) return e;
    }
    count_launch();
    return cudaGetLastError();
}

template <int BN, int NPASS, int CG, bool SPL, bool F16 = false>
cudaError_t dispatch_epi(int epi, const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                         const CUtensorMap& bl, const GemmParams& p, int num_sms, cudaStream_t s) {
    switch (epi) {
        case EPI_STORE: return launch_inst<BN, NPASS, EPI_STORE, CG, SPL, F16>(ah, al, bh, bl, p, num_sms, s);
        case EPI_SYM_EMA: return launch_inst<BN, NPASS, EPI_SYM_EMA, CG, SPL, F16>(ah, al, bh, bl, p, num_sms, s);
        case EPI_SPLIT: return launch_inst<BN, NPASS, EPI_SPLIT, CG, SPL, F16>(ah, al, bh, bl, p, num_sms, s);
        case EPI_SPLIT_T: return launch_inst<BN, NPASS, EPI_SPLIT_T, CG, SPL, F16>(ah, al, bh, bl, p, num_sms, s);
        case EPI_ADAM: return launch_inst<BN, NPASS, EPI_ADAM, CG, SPL, F16>(ah, al, bh, bl, p, num_sms, s);
        case EPI_APPLY: return launch_inst<BN, NPASS, EPI_APPLY, CG, SPL, F16>(ah, al, bh, bl, p, num_sms, s);
        case EPI_SYM_SPLIT: return launch_inst<BN, NPASS, EPI_SYM_SPLIT, CG, SPL, F16>(ah, al, bh, bl, p, num_sms, s);
        case EPI_NS: return launch_inst<BN, NPASS, EPI_NS, CG, SPL, F16>(ah, al, bh, bl, p, num_sms, s);
        case EPI_SPLIT2: return launch_inst<BN, NPASS, EPI_SPLIT2, CG, SPL, F16>(ah, al, bh, bl, p, num_sms, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

int gemm_bn_for(int n, int batch) {
    static const int force = getenv("ASG_GEMM_BN") ? atoi(getenv("ASG_GEMM_BN")) : 0;  // tuning experiments
    if (force == 128) return 128;
    if (n % 256 != 0) return 128;
    // symmetric outputs of a few matrices (C1: one 1024^2 block): the 256-wide CTA-pair
    // triangle (10 tiles at 1024) would leave most SMs idle; 128-wide tiles give 36
    const int t = n / 256;
    return int64_t(batch) * t * (t + 1) / 2 < 74 ? 128 : 256;
}

int gemm_sym_tile_list(int n, int bn, int2* out) {
    int count = 0;
    for (int tm = 0; tm < n / 128; ++tm)
        for (int tn = 0; tn < n / bn; ++tn)
            if ((tm + 1) * 128 - 1 >= tn * bn) {
                if (out) out[count] = make_int2(tm, tn);
                ++count;
            }
    return count;
}

// CTA-pair (cta_group::2, 256-row tiles) schedules: on unless ASG_GEMM_PAIR=0.
static bool pair_enabled() {
    static const bool on = !(getenv("ASG_GEMM_PAIR") && atoi(getenv("ASG_GEMM_PAIR")) == 0);
    return on;
}

cudaError_t gemm_launch(const GemmLaunch& g, int precision, int num_sms, cudaStream_t stream) {
    const int M = g.A.rows, N = g.B.rows, K = g.A.K;
    if (M % 128 || N % 128 || K % 32 || g.B.K != K) return cudaErrorInvalidValue;
    // symmetric schedules: the tile width their list was built for (gemm_bn_for(N, batch) of
    // the owner; the 128-wide lower triangle has more tiles than the 256-wide one)
    int bn = (N % 256 == 0) ? 256 : 128;
    if (g.sym_tiles && bn == 256 && g.sym_tiles_count == gemm_sym_tile_list(N, 128, nullptr)) bn = 128;
    // Small rectangular problems: 128-wide tiles when 256-wide ones would not
    // fill two waves of the persistent grid (symmetric schedules keep the tile
    // width their tile lists were built for).
    if (!g.sym_tiles && bn == 256 && int64_t(g.batch) * (M / 128) * (N / 256) < 2 * int64_t(num_sms)) bn = 128;
    // CTA pairs: 256 x BN tiles, when M splits into 256-row tiles, the pair grid
    // still gets two waves, and (symmetric outputs) the 256 x 256 lower-triangle
    // grid covers the output (N % 256 == 0, M == N)
    bool pair = pair_enabled() && M % 256 == 0;
    if (pair && g.sym_tiles) pair = (bn == 256 && M == N);
    if (pair && !g.sym_tiles && int64_t(g.batch) * (M / 256) * (N / bn) < int64_t(num_sms)) pair = false;
    const int tm_rows = pair ? 256 : 128;
    const int brows = pair ? bn / 2 : bn;
    const bool split = precision != ASG_PREC_TF32;  // 3XTF32, 3XTF32_SMEM, 3XF16
    // 3xFP16: both operands fp16 (hi, lo) pairs with per-batch scales
    const bool f16 = g.A.scale != nullptr;
    if (f16 != (g.B.scale != nullptr) || (f16 && (!g.A.lo || !g.B.lo || !split)))
        return cudaErrorInvalidValue;
    // 3xTF32 operands without a lo array hold plain fp32: split in shared memory (SPL)
    const bool a_raw = split && !f16 && !g.A.lo, b_raw = split && !f16 && !g.B.lo;
    const bool spl = a_raw || b_raw;
    CUtensorMap ah, al, bh, bl;
    if (!make_map(&ah, g.A.hi, K, M, g.batch, 128, f16)) return cudaErrorInvalidValue;
    if (!make_map(&bh, g.B.hi, K, N, g.batch, brows, f16)) return cudaErrorInvalidValue;
    al = ah;
    bl = bh;
    if (split && !a_raw && !make_map(&al, g.A.lo, K, M, g.batch, 128, f16)) return cudaErrorInvalidValue;
    if (split && !b_raw && !make_map(&bl, g.B.lo, K, N, g.batch, brows, f16)) return cudaErrorInvalidValue;
    GemmParams p = g.p;
    p.raw_out = split ? 1 : 0;
    p.a_raw = a_raw ? 1 : 0;
    p.b_raw = b_raw ? 1 : 0;
    p.ascale = g.A.scale;
    p.bscale = g.B.scale;
    p.M = M;
    p.N = N;
    p.K = K;
    p.batch = g.batch;
    p.tiles_n = N / bn;
    p.sym_T = 0;
    static const int raster = getenv("ASG_GEMM_RASTER") ? atoi(getenv("ASG_GEMM_RASTER")) : 0;  // tuning
    p.raster = raster;
    if (g.sym_tiles && pair) {
        const int T = N / 256;
        p.tile_list = nullptr;
        p.sym_T = T;
        p.tiles_per_batch = T * (T + 1) / 2;
    } else if (g.sym_tiles) {
        p.tile_list = g.sym_tiles;
        p.tiles_per_batch = g.sym_tiles_count;
    } else {
        p.tile_list = nullptr;
        p.tiles_per_batch = (M / tm_rows) * (N / bn);
    }
    p.num_tiles = p.tiles_per_batch * g.batch;
    if (f16) {
        if (pair)
            return bn == 256 ? dispatch_epi<256, 3, 2, false, true>(g.epi, ah, al, bh, bl, p, num_sms, stream)
                             : dispatch_epi<128, 3, 2, false, true>(g.epi, ah, al, bh, bl, p, num_sms, stream);
        return bn == 256 ? dispatch_epi<256, 3, 1, false, true>(g.epi, ah, al, bh, bl, p, num_sms, stream)
                         : dispatch_epi<128, 3, 1, false, true>(g.epi, ah, al, bh, bl, p, num_sms, stream);
    }
    if (spl) {
        if (pair)
            return bn == 256 ? dispatch_epi<256, 3, 2, true>(g.epi, ah, al, bh, bl, p, num_sms, stream)
                             : dispatch_epi<128, 3, 2, true>(g.epi, ah, al, bh, bl, p, num_sms, stream);
        return bn == 256 ? dispatch_epi<256, 3, 1, true>(g.epi, ah, al, bh, bl, p, num_sms, stream)
                         : dispatch_epi<128, 3, 1, true>(g.epi, ah, al, bh, bl, p, num_sms, stream);
    }
    if (pair) {
        if (bn == 256)
            return split ? dispatch_epi<256, 3, 2, false>(g.epi, ah, al, bh, bl, p, num_sms, stream)
                         : dispatch_epi<256, 1, 2, false>(g.epi, ah, al, bh, bl, p, num_sms, stream);
        return split ? dispatch_epi<128, 3, 2, false>(g.epi, ah, al, bh, bl, p, num_sms, stream)
                     : dispatch_epi<128, 1, 2, false>(g.epi, ah, al, bh, bl, p, num_sms, stream);
    }
    if (bn == 256)
        return split ? dispatch_epi<256, 3, 1, false>(g.epi, ah, al, bh, bl, p, num_sms, stream)
                     : dispatch_epi<256, 1, 1, false>(g.epi, ah, al, bh, bl, p, num_sms, stream);
    return split ? dispatch_epi<128, 3, 1, false>(g.epi, ah, al, bh, bl, p, num_sms, stream)
                 : dispatch_epi<128, 1, 1, false>(g.epi, ah, al, bh, bl, p, num_sms, stream);
}

// ============================================================================
// K1: gradient prep
// ============================================================================
__global__ void prep_grad_kernel(const BlockRef* __restrict__ blocks, int M, int N,
                                 const float* __restrict__ scale_dev, float scale_val,
                                 float* __restrict__ Gh, float* __restrict__ Gl,
                                 float* __restrict__ GTh, float* __restrict__ GTl) {
    __shared__ float th[32][33];
    __shared__ float tl[32][33];
    const int b = blockIdx.z;
    const BlockRef blk = blocks[b];
    const float s = scale_dev ? *scale_dev : scale_val;
    const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    const int64_t slab = int64_t(M) * N;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int i = i0 + dy, j = j0 + threadIdx.x;
        float x = 0.f;
        if (i < blk.rows && j < blk.cols) x = s * blk.src[int64_t(i) * blk.ld + j];
        float h, l;
        if (Gl) {
            split_tf32(x, h, l);
        } else {
            h = x;
            l = 0.f;
        }
        Gh[b * slab + int64_t(i) * N + j] = h;
        if (Gl) Gl[b * slab + int64_t(i) * N + j] = l;
        th[dy][threadIdx.x] = h;
        tl[dy][threadIdx.x] = l;
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int jj = j0 + dy, ii = i0 + threadIdx.x;  // GT[jj][ii] = G[ii][jj]
        GTh[b * slab + int64_t(jj) * M + ii] = th[threadIdx.x][dy];
        if (GTl) GTl[b * slab + int64_t(jj) * M + ii] = tl[threadIdx.x][dy];
    }
}

// 64 x 64 tiles, float4 accesses (blocks with 16-byte aligned rows: every
// column offset, leading dimension and block width a multiple of 4).
__global__ void __launch_bounds__(256) prep_grad_vec_kernel(const BlockRef* __restrict__ blocks, int M, int N,
                                                            const float* __restrict__ scale_dev, float scale_val,
                                                            float* __restrict__ Gh, float* __restrict__ Gl,
                                                            float* __restrict__ GTh, float* __restrict__ GTl) {
    __shared__ float th[64][65];
    __shared__ float tl[64][65];
    const int b = blockIdx.z;
    const BlockRef blk = blocks[b];
    const float s = scale_dev ? *scale_dev : scale_val;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 16 x 16
    const int j0 = blockIdx.x * 64, i0 = blockIdx.y * 64;
    const int64_t slab = int64_t(M) * N;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int i = i0 + ty + 16 * r, j = j0 + tx * 4;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < blk.rows && j < blk.cols) x = *reinterpret_cast<const float4*>(blk.src + int64_t(i) * blk.ld + j);
        float4 h, l;
        split_tf32(s * x.x, h.x, l.x);
        split_tf32(s * x.y, h.y, l.y);
        split_tf32(s * x.z, h.z, l.z);
        split_tf32(s * x.w, h.w, l.w);
        if (!Gl) h = make_float4(s * x.x, s * x.y, s * x.z, s * x.w);
        *reinterpret_cast<float4*>(Gh + b * slab + int64_t(i) * N + j) = h;
        if (Gl) *reinterpret_cast<float4*>(Gl + b * slab + int64_t(i) * N + j) = l;
        const int rr = ty + 16 * r, cc = tx * 4;
        th[rr][cc] = h.x;
        th[rr][cc + 1] = h.y;
        th[rr][cc + 2] = h.z;
        th[rr][cc + 3] = h.w;
        tl[rr][cc] = l.x;
        tl[rr][cc + 1] = l.y;
        tl[rr][cc + 2] = l.z;
        tl[rr][cc + 3] = l.w;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int jj = j0 + ty + 16 * r, ii = i0 + tx * 4;  // GT[jj][ii..ii+3] = G[ii..ii+3][jj]
        const int cj = ty + 16 * r, ri = tx * 4;
        *reinterpret_cast<float4*>(GTh + b * slab + int64_t(jj) * M + ii) =
            make_float4(th[ri][cj], th[ri + 1][cj], th[ri + 2][cj], th[ri + 3][cj]);
        if (GTl)
            *reinterpret_cast<float4*>(GTl + b * slab + int64_t(jj) * M + ii) =
                make_float4(tl[ri][cj], tl[ri + 1][cj], tl[ri + 2][cj], tl[ri + 3][cj]);
    }
}

void launch_prep_grad(const BlockRef* blocks_dev, int nb, int M, int N, const float* scale_dev,
                      float scale_val, float* Gh, float* Gl, float* GTh, float* GTl, cudaStream_t s, bool vec) {
    if (vec) {
        dim3 grid(N / 64, M / 64, nb), block(16, 16);
        prep_grad_vec_kernel<<<grid, block, 0, s>>>(blocks_dev, M, N, scale_dev, scale_val, Gh, Gl, GTh, GTl);
    } else {
        dim3 grid(N / 32, M / 32, nb), block(32, 8);
        prep_grad_kernel<<<grid, block, 0, s>>>(blocks_dev, M, N, scale_dev, scale_val, Gh, Gl, GTh, GTl);
    }
    count_launch();
}

__global__ void identity_split_kernel(float* hi, float* lo, int M, int m) {
    const int64_t b = blockIdx.y;
    const int64_t slab = int64_t(M) * M;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < slab; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(uint32_t(e) / uint32_t(M)), j = int(uint32_t(e) - uint32_t(i) * uint32_t(M));  // per-matrix index < 2^31
        hi[b * slab + e] = (i == j && i < m) ? 1.f : 0.f;
        if (lo) lo[b * slab + e] = 0.f;
    }
}

void launch_identity_split(float* hi, float* lo, int nb, int M, int m, cudaStream_t s) {
    identity_split_kernel<<<dim3(256, nb), 256, 0, s>>>(hi, lo, M, m);
    count_launch();
}

__global__ void identity_f32_kernel(float* a, int M, int m, float diag) {
    const int64_t b = blockIdx.y;
    const int64_t slab = int64_t(M) * M;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < slab; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(uint32_t(e) / uint32_t(M)), j = int(uint32_t(e) - uint32_t(i) * uint32_t(M));  // per-matrix index < 2^31
        a[b * slab + e] = (i == j && i < m) ? diag : 0.f;
    }
}

void launch_identity_f32(float* a, int nb, int M, int m, float diag, cudaStream_t s) {
    identity_f32_kernel<<<dim3(256, nb), 256, 0, s>>>(a, M, m, diag);
    count_launch();
}

// ============================================================================
// K10: global squared norm + non-finite flag; clip scale
// ============================================================================
__global__ void sqnorm_kernel(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                              double* acc, int* flag) {
    double s = 0.0;
    bool bad = false;
    const int64_t n = rows * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const float v = x[(e / cols) * ld + (e % cols)];
        bad |= !isfinite(v);
        s += double(v) * double(v);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
    __shared__ double red[32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = s;
    __syncthreads();
    if (w == 0) {
        s = (l < int(blockDim.x >> 5)) ? red[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
        if (l == 0) atomicAdd(acc, s);
    }
    if (bad && flag) atomicOr(flag, 1);
}

void launch_sqnorm(const float* x, int64_t rows, int64_t cols, int64_t ld, double* acc, int* flag,
                   cudaStream_t s) {
    const int64_t n = rows * cols;
    int grid = int((n + 1023) / 1024);
    if (grid > 1184) grid = 1184;
    if (grid < 1) grid = 1;
    sqnorm_kernel<<<grid, 256, 0, s>>>(x, rows, cols, ld, acc, flag);
    count_launch();
}

// Multi-tensor sum of squares: one CTA per chunk of one tensor.
__global__ void sqnorm_multi_kernel(const SqChunk* __restrict__ chunks, double* acc, int* flag) {
    const SqChunk c = chunks[blockIdx.x];
    double s = 0.0;
    bool bad = false;
    const float* base = c.x + c.e0;
    const int64_t n = c.e1 - c.e0;
    if (c.ld == c.cols && (reinterpret_cast<uintptr_t>(base) & 15) == 0 && (n & 3) == 0) {
        // contiguous chunk: 16-byte loads, no index arithmetic per element
        const float4* b4 = reinterpret_cast<const float4*>(base);
        for (int64_t i = threadIdx.x; i < n / 4; i += blockDim.x) {
            const float4 v = __ldcs(b4 + i);
            bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
            s += double(v.x) * double(v.x) + double(v.y) * double(v.y) + double(v.z) * double(v.z) +
                 double(v.w) * double(v.w);
        }
    } else {
        for (int64_t e = c.e0 + threadIdx.x; e < c.e1; e += blockDim.x) {
            const float v = c.x[(e / c.cols) * c.ld + (e % c.cols)];
            bad |= !isfinite(v);
            s += double(v) * double(v);
        }
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
    __shared__ double red[32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = s;
    __syncthreads();
    if (w == 0) {
        s = (l < int(blockDim.x >> 5)) ? red[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
        if (l == 0) atomicAdd(acc, s);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, 1);
}

void launch_sqnorm_multi(const SqChunk* chunks, int count, double* acc, int* flag, cudaStream_t s) {
    if (count <= 0) return;
    sqnorm_multi_kernel<<<count, 256, 0, s>>>(chunks, acc, flag);
    count_launch();
}

__global__ void clip_scale_kernel(const double* sq, double clip, float* out) {
    const double norm = sqrt(*sq);
    *out = (norm <= clip || norm == 0.0) ? 1.f : float(clip / norm);
}

void launch_clip_scale(const double* sqnorm, double clip_norm, float* scale_out, cudaStream_t s) {
    clip_scale_kernel<<<1, 1, 0, s>>>(sqnorm, clip_norm, scale_out);
    count_launch();
}

// ============================================================================
// K9: AdamW + apply (1-D parameters)
// ============================================================================
__global__ void adamw_apply_kernel(float* __restrict__ theta, int64_t ld_t, const float* __restrict__ grad,
                                   int64_t ld_g, int64_t rows, int64_t cols, float* __restrict__ m,
                                   float* __restrict__ v, const float* scale_dev, float scale_val, float b1,
                                   float b2, float inv_bc1, float inv_bc2, float eps, float lr_eff, float wd,
                                   int* flag) {
    const float s = scale_dev ? *scale_dev : scale_val;
    const int64_t n = rows * cols;
    bool bad = false;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / cols, c = e % cols;
        const float g = s * grad[r * ld_g + c];
        bad |= !isfinite(g);
        const float mm = b1 * m[e] + (1.f - b1) * g;
        const float vv = b2 * v[e] + (1.f - b2) * g * g;
        m[e] = mm;
        v[e] = vv;
        const float u = (mm * inv_bc1) / (sqrtf(vv * inv_bc2) + eps);
        float& t = theta[r * ld_t + c];
        t = t - lr_eff * (u + wd * t);
    }
    if (bad && flag) atomicOr(flag, 1);
}

void launch_adamw_apply(float* theta, int64_t ld_t, const float* grad, int64_t ld_g, int64_t rows, int64_t cols,
                        float* m, float* v, const float* scale_dev, float scale_val, float b1, float b2,
                        float inv_bc1, float inv_bc2, float eps, float lr_eff, float wd, int* flag,
                        cudaStream_t s) {
    const int64_t n = rows * cols;
    int grid = int((n + 255) / 256);
    if (grid > 1184) grid = 1184;
    if (grid < 1) grid = 1;
    adamw_apply_kernel<<<grid, 256, 0, s>>>(theta, ld_t, grad, ld_g, rows, cols, m, v, scale_dev, scale_val, b1,
                                            b2, inv_bc1, inv_bc2, eps, lr_eff, wd, flag);
}

// Multi-tensor AdamW + apply: every 1-D / degenerate parameter of the step in
// one launch (blockIdx.y = parameter).
__global__ void adamw_multi_kernel(const AdamEntry* __restrict__ entries, float scale_val, float b1, float b2,
                                   float inv_bc1, float inv_bc2, float eps, float lr_eff, float wd, int* flag) {
    const AdamEntry en = entries[blockIdx.y];
    const int64_t n = en.rows * en.cols;
    bool bad = false;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / en.cols, c = e % en.cols;
        const float g = scale_val * en.grad[r * en.ld_g + c];
        if (!isfinite(g)) {  // adamw_step throws NonFinite before touching state (precond.cpp:231)
            bad = true;
            continue;
        }
        const float mm = b1 * en.m[e] + (1.f - b1) * g;
        const float vv = b2 * en.v[e] + (1.f - b2) * g * g;
        en.m[e] = mm;
        en.v[e] = vv;
        const float u = (mm * inv_bc1) / (sqrtf(vv * inv_bc2) + eps);
        float& t = en.theta[r * en.ld_t + c];
        t = t - lr_eff * (u + wd * t);
    }
    if (bad && flag) atomicOr(flag, 1);
}

void launch_adamw_multi(const AdamEntry* entries, int count, int64_t max_elems, float scale_val, float b1, float b2,
                        float inv_bc1, float inv_bc2, float eps, float lr_eff, float wd, int* flag, cudaStream_t s) {
    if (count <= 0) return;
    int gx = int((max_elems + 255) / 256);
    if (gx > 64) gx = 64;
    if (gx < 1) gx = 1;
    adamw_multi_kernel<<<dim3(gx, count), 256, 0, s>>>(entries, scale_val, b1, b2, inv_bc1, inv_bc2, eps, lr_eff, wd,
                                                       flag);
    count_launch();
}

// ============================================================================
// K8: snapshot (fp32 factor slab -> fp64 shadow)
// ============================================================================
__global__ void snapshot_kernel(const float* __restrict__ src, int M, int m, double* __restrict__ dst) {
    const int64_t b = blockIdx.y;
    const int64_t n = int64_t(m) * m;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(uint32_t(e) / uint32_t(m)), j = int(uint32_t(e) - uint32_t(i) * uint32_t(m));  // per-matrix index < 2^31
        dst[b * n + e] = double(src[b * int64_t(M) * M + int64_t(i) * M + j]);
    }
}

void launch_snapshot(const float* src, int nb, int M, int m, double* dst, cudaStream_t s) {
    snapshot_kernel<<<dim3(128, nb), 256, 0, s>>>(src, M, m, dst);
    count_launch();
}

// ============================================================================
// K6: batched symmetric eigendecomposition (fp64)
//
// One CTA per matrix; parallel (round-robin tournament) two-sided Jacobi on
// the matrix held in global memory (L2-resident for the dims this kernel is
// used at). Same stopping rule as the reference's cyclic Jacobi: off-diagonal
// Frobenius norm <= 1e-12 * ||A||_F within 30 sweeps (densela.hpp:192-249),
// values ascending by a stable index-ordered rank (densela.hpp:251-262).
// ============================================================================
namespace {
constexpr int kEigThreads = 512;
constexpr int kMaxEigN = 4096;

__device__ double block_reduce_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = (l < int(blockDim.x >> 5)) ? red[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
        if (l == 0) red[0] = v;
    }
    __syncthreads();
    const double r = red[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ int tourney(int pos, int r, int P) { return pos == 0 ? 0 : 1 + (pos - 1 + r) % (P - 1); }
}  // namespace

__global__ void __launch_bounds__(kEigThreads) sym_eig_kernel(const double* __restrict__ Ain, double* values,
                                                              double* vectors, double* work, int n, int* status) {
    extern __shared__ double sh[];
    double* cs = sh;                 // [P/2] cosines
    double* sn = cs + kMaxEigN / 2;  // [P/2] sines
    __shared__ double red[32];
    const int64_t b = blockIdx.x;
    const int64_t nn = int64_t(n) * n;
    const double* A0 = Ain + b * nn;
    double* A = work + b * nn;
    double* V = vectors + b * nn;
    const int tid = threadIdx.x, nt = blockDim.x;

    double fro = 0.0;
    bool bad = false;
    for (int64_t e = tid; e < nn; e += nt) {
        const double x = A0[e];
        bad |= !isfinite(x);
        A[e] = x;
        V[e] = (e / n == e % n) ? 1.0 : 0.0;
        fro += x * x;
    }
    const int any_bad = __syncthreads_or(bad);
    if (any_bad) {
        if (tid == 0) atomicCAS(&status[b], ASG_OK, ASG_ERR_NON_FINITE);
        return;
    }
    fro = sqrt(block_reduce_sum(fro, red));
    const double tol = 1e-12 * fro;
    const int P = n + (n & 1);  // players (a dummy when n is odd)
    const int half = P / 2;

    auto off_norm = [&]() {
        double acc = 0.0;
        for (int64_t e = tid; e < nn; e += nt) {
            const int i = int(uint32_t(e) / uint32_t(n)), j = int(uint32_t(e) - uint32_t(i) * uint32_t(n));  // per-matrix index < 2^31
            if (j > i) acc += A[e] * A[e];
        }
        return sqrt(2.0 * block_reduce_sum(acc, red));
    };

    bool converged = (n <= 1) || off_norm() <= tol;
    for (int sweep = 0; sweep < 30 && !converged; ++sweep) {
        for (int r = 0; r < P - 1; ++r) {
            // rotation parameters for every pair of this round
            for (int k = tid; k < half; k += nt) {
                int p = tourney(k, r, P), q = tourney(P - 1 - k, r, P);
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                double c = 1.0, s = 0.0;
                if (q < n) {
                    const double apq = A[int64_t(p) * n + q];
                    if (apq != 0.0) {
                        const double app = A[int64_t(p) * n + p], aqq = A[int64_t(q) * n + q];
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                                      : -1.0 / (-tau + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                    }
                }
                cs[k] = c;
                sn[k] = s;
            }
            __syncthreads();
            // rows: A <- J^T A
            for (int64_t e = tid; e < int64_t(half) * n; e += nt) {
                const int k = int(e / n), j = int(e % n);
                const double s = sn[k];
                if (s == 0.0) continue;
                int p = tourney(k, r, P), q = tourney(P - 1 - k, r, P);
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                const double c = cs[k];
                const double x = A[int64_t(p) * n + j], y = A[int64_t(q) * n + j];
                A[int64_t(p) * n + j] = c * x - s * y;
                A[int64_t(q) * n + j] = s * x + c * y;
            }
            __syncthreads();
            // columns: A <- A J, V <- V J
            for (int64_t e = tid; e < int64_t(half) * n; e += nt) {
                const int k = int(e % half), i = int(e / half);
                const double s = sn[k];
                if (s == 0.0) continue;
                int p = tourney(k, r, P), q = tourney(P - 1 - k, r, P);
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                const double c = cs[k];
                double x = A[int64_t(i) * n + p], y = A[int64_t(i) * n + q];
                double np = c * x - s * y, nq = s * x + c * y;
                if (i == p) nq = 0.0;  // exact zero in the rotated plane
                if (i == q) np = 0.0;
                A[int64_t(i) * n + p] = np;
                A[int64_t(i) * n + q] = nq;
                x = V[int64_t(i) * n + p];
                y = V[int64_t(i) * n + q];
                V[int64_t(i) * n + p] = c * x - s * y;
                V[int64_t(i) * n + q] = s * x + c * y;
            }
            __syncthreads();
        }
        converged = off_norm() <= tol;
    }
    if (!converged) {
        if (tid == 0) atomicCAS(&status[b], ASG_OK, ASG_ERR_NO_CONVERGENCE);
        return;
    }
    // ascending stable order by rank; diag -> shared, permuted vectors -> work
    double* d = sh;  // reuse: n <= kMaxEigN doubles
    __syncthreads();
    for (int i = tid; i < n; i += nt) d[i] = A[int64_t(i) * n + i];
    __syncthreads();
    for (int i = tid; i < n; i += nt) {
        const double di = d[i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double dj = d[j];
            rank += (dj < di) || (dj == di && j < i);
        }
        values[b * n + rank] = di;
        for (int row = 0; row < n; ++row) A[int64_t(row) * n + rank] = V[int64_t(row) * n + i];
    }
    __syncthreads();
    for (int64_t e = tid; e < nn; e += nt) V[e] = A[e];
}

void launch_sym_eig(const double* A, double* values, double* vectors, double* work, int nb, int n, int* status,
                    cudaStream_t s) {
    static std::atomic<uint64_t> attr_bits{0};
    const size_t smem = sizeof(double) * kMaxEigN;
    if (first_on_device(attr_bits)) {
        cudaFuncSetAttribute(sym_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    }
    sym_eig_kernel<<<nb, kEigThreads, smem, s>>>(A, values, vectors, work, n, status);
    count_launch();
}

// ============================================================================
// K6: damping, column scaling (roots), conversions
// ============================================================================
__global__ void relative_damping_kernel(const double* A, int n, double damping, double* eps) {
    __shared__ double red[32];
    const int64_t b = blockIdx.x;
    double tr = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) tr += A[b * int64_t(n) * n + int64_t(i) * n + i];
    tr = block_reduce_sum(tr, red);
    if (threadIdx.x == 0) eps[b] = n > 0 ? damping * tr / double(n) : 0.0;
}

void launch_relative_damping(const double* A, int nb, int n, double damping, double* eps, cudaStream_t s) {
    relative_damping_kernel<<<nb, 256, 0, s>>>(A, n, damping, eps);
    count_launch();
}

__global__ void scale_columns_kernel(const double* V, const double* values, const double* eps, double power,
                                     int n, double* W, int* status) {
    const int64_t b = blockIdx.y;
    const int64_t nn = int64_t(n) * n;
    const double e = eps ? eps[b] : 0.0;
    // The factor is fp32 (accumulated on tensor cores): eigenvalues within its
    // rounding level, |lam| <= 4 * 2^-24 * n * max|lam|, are numerically zero.
    // Negative ones in that band are clamped to 0 before damping; only a damped
    // eigenvalue that is still <= 0 is NotPsd (densela.hpp:274-278).
    const double lam_abs = fmax(fabs(values[b * n]), fabs(values[b * n + n - 1]));
    const double tau = 4.0 * 5.9604644775390625e-08 * double(n) * lam_abs;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < nn; idx += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(idx % n);
        double lam = values[b * n + j];
        if (lam < 0.0 && lam >= -tau) lam = 0.0;
        const double damped = lam + e;
        if (damped <= 0.0) {
            atomicCAS(&status[b], ASG_OK, ASG_ERR_NOT_PSD);
            W[b * nn + idx] = 0.0;
            continue;
        }
        W[b * nn + idx] = V[b * nn + idx] * pow(damped, power);
    }
}

void launch_scale_columns(const double* V, const double* values, const double* eps, double power, int nb, int n,
                          double* W, int* status, cudaStream_t s) {
    scale_columns_kernel<<<dim3(128, nb), 256, 0, s>>>(V, values, eps, power, n, W, status);
    count_launch();
}

// fp64 tiled batched GEMM on CUDA cores (64 x 64 tiles, 4 x 4 per thread).
__global__ void dgemm_kernel(bool ta, bool tb, int m, int n, int k, double alpha, const double* __restrict__ A,
                             int64_t lda, int64_t sa, const double* __restrict__ B, int64_t ldb, int64_t sb,
                             double beta, double* __restrict__ C, int64_t ldc, int64_t sc) {
    __shared__ double As[16][65];
    __shared__ double Bs[16][65];
    const int64_t bz = blockIdx.z;
    A += bz * sa;
    B += bz * sb;
    C += bz * sc;
    const int row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < k; k0 += 16) {
        for (int e = threadIdx.x; e < 16 * 64; e += 256) {
            const int kk = e / 64, rr = e % 64;
            const int gr = row0 + rr, gk = k0 + kk;
            double a = 0.0;
            if (gr < m && gk < k) a = ta ? A[int64_t(gk) * lda + gr] : A[int64_t(gr) * lda + gk];
            As[kk][rr] = a;
            const int gc = col0 + rr;
            double bv = 0.0;
            if (gc < n && gk < k) bv = tb ? B[int64_t(gc) * ldb + gk] : B[int64_t(gk) * ldb + gc];
            Bs[kk][rr] = bv;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            double a[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = row0 + ty * 4 + i, c = col0 + tx * 4 + j;
            if (r < m && c < n) {
                double v = alpha * acc[i][j];
                if (beta != 0.0) v += beta * C[int64_t(r) * ldc + c];
                C[int64_t(r) * ldc + c] = v;
            }
        }
}

void launch_dgemm(bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int64_t lda, int64_t sa,
                  const double* B, int64_t ldb, int64_t sb, double beta, double* C, int64_t ldc, int64_t sc, int nb,
                  cudaStream_t s) {
    dim3 grid((n + 63) / 64, (m + 63) / 64, nb);
    dgemm_kernel<<<grid, 256, 0, s>>>(ta, tb, m, n, k, alpha, A, lda, sa, B, ldb, sb, beta, C, ldc, sc);
    count_launch();
}

__global__ void f64_to_split_kernel(const double* __restrict__ src, int n, int M, bool sym, float* hi, float* lo,
                                    float* hi_t, float* lo_t) {
    __shared__ float th[32][33];
    __shared__ float tl[32][33];
    const int64_t b = blockIdx.z;
    const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    const int64_t slab = int64_t(M) * M, nn = int64_t(n) * n;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int i = i0 + dy, j = j0 + threadIdx.x;
        double x = 0.0;
        if (i < n && j < n) {
            x = src[b * nn + int64_t(i) * n + j];
            if (sym) x = 0.5 * (x + src[b * nn + int64_t(j) * n + i]);
        }
        const float xf = float(x);
        float h = xf, l = 0.f;
        if (lo) {
            // hi/lo from the fp64 value: hi = tf32(x), lo = tf32(x - hi)
            h = tf32_round(xf);
            l = tf32_round(float(x - double(h)));
        }
        hi[b * slab + int64_t(i) * M + j] = h;
        if (lo) lo[b * slab + int64_t(i) * M + j] = l;
        th[dy][threadIdx.x] = h;
        tl[dy][threadIdx.x] = l;
    }
    if (!hi_t) return;
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int jj = j0 + dy, ii = i0 + threadIdx.x;
        hi_t[b * slab + int64_t(jj) * M + ii] = th[threadIdx.x][dy];
        if (lo_t) lo_t[b * slab + int64_t(jj) * M + ii] = tl[threadIdx.x][dy];
    }
}

void launch_f64_to_split(const double* src, int nb, int n, int M, bool symmetrize, float* hi, float* lo,
                         float* hi_t, float* lo_t, cudaStream_t s) {
    dim3 grid(M / 32, M / 32, nb), block(32, 8);
    f64_to_split_kernel<<<grid, block, 0, s>>>(src, n, M, symmetrize, hi, lo, hi_t, lo_t);
    count_launch();
}

__global__ void f64_to_f32_kernel(const double* src, int rows, int cols, float* dst, int R, int Cc) {
    const int64_t b = blockIdx.y;
    const int64_t tot = int64_t(R) * Cc;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(uint32_t(e) / uint32_t(Cc)), j = int(uint32_t(e) - uint32_t(i) * uint32_t(Cc));  // per-matrix index < 2^31
        dst[b * tot + e] = (i < rows && j < cols) ? float(src[b * int64_t(rows) * cols + int64_t(i) * cols + j]) : 0.f;
    }
}

void launch_f64_to_f32(const double* src, int nb, int rows, int cols, float* dst, int R, int Cc, cudaStream_t s) {
    f64_to_f32_kernel<<<dim3(128, nb), 256, 0, s>>>(src, rows, cols, dst, R, Cc);
    count_launch();
}

__global__ void f32_to_f64_kernel(const float* src, int rows, int cols, int R, int Cc, double* dst) {
    const int64_t b = blockIdx.y;
    const int64_t tot = int64_t(rows) * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < tot; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(uint32_t(e) / uint32_t(cols)), j = int(uint32_t(e) - uint32_t(i) * uint32_t(cols));  // per-matrix index < 2^31
        dst[b * tot + e] = double(src[b * int64_t(R) * Cc + int64_t(i) * Cc + j]);
    }
}

void launch_f32_to_f64(const float* src, int nb, int rows, int cols, int R, int Cc, double* dst, cudaStream_t s) {
    f32_to_f64_kernel<<<dim3(128, nb), 256, 0, s>>>(src, rows, cols, R, Cc, dst);
    count_launch();
}

__global__ void square_f64_kernel(const double* a, double* out, int64_t n) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
        out[e] = a[e] * a[e];
}

void launch_square_f64(const double* a, double* out, int64_t n, cudaStream_t s) {
    square_f64_kernel<<<256, 256, 0, s>>>(a, out, n);
    count_launch();
}

// ============================================================================
// fp32-level refresh (tensor-core transforms): split / transpose / scale
// ============================================================================
__global__ void merge_pair_kernel(const float* __restrict__ hi, const float* __restrict__ lo, float* __restrict__ dst,
                                  int64_t count) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x)
        dst[e] = hi[e] + lo[e];
}

void launch_merge_pair(const float* hi, const float* lo, float* dst, int64_t count, cudaStream_t s) {
    const int64_t blocks = (count + 255) / 256;
    merge_pair_kernel<<<int(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(hi, lo, dst, count);
    count_launch();
}

__global__ void split_slab_kernel(const float* __restrict__ src, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t count) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x) {
        float h, l;
        split_tf32(src[e], h, l);
        hi[e] = h;
        lo[e] = l;
    }
}

void launch_split_slab(const float* src, float* hi, float* lo, int64_t count, cudaStream_t s) {
    split_slab_kernel<<<1184, 256, 0, s>>>(src, hi, lo, count);
    count_launch();
}

// [b][M][M] fp32 slab (leading m x m) -> [b][m][m] fp64, symmetrized.
__global__ void snapshot_sym_kernel(const float* __restrict__ src, int M, int m, double* __restrict__ dst) {
    const int64_t b = blockIdx.y;
    const int64_t n = int64_t(m) * m;
    const float* sb = src + b * int64_t(M) * M;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(uint32_t(e) / uint32_t(m)), j = int(uint32_t(e) - uint32_t(i) * uint32_t(m));  // per-matrix index < 2^31
        dst[b * n + e] = 0.5 * (double(sb[int64_t(i) * M + j]) + double(sb[int64_t(j) * M + i]));
    }
}

void launch_snapshot_sym(const float* src, int nb, int M, int m, double* dst, cudaStream_t s) {
    snapshot_sym_kernel<<<dim3(128, nb), 256, 0, s>>>(src, M, m, dst);
    count_launch();
}

// dst[b][c][r] = split(src_hi[b][r][c] + src_lo[b][r][c]); R, C multiples of 32.
__global__ void transpose_split_kernel(const float* __restrict__ src_hi, const float* __restrict__ src_lo, int R, int C,
                                       float* __restrict__ dst_hi, float* __restrict__ dst_lo, int square) {
    __shared__ float t[32][33];
    const int64_t b = blockIdx.z;
    const int64_t slab = int64_t(R) * C;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t off = b * slab + int64_t(r0 + dy) * C + c0 + threadIdx.x;
        float x = src_hi[off] + (src_lo ? src_lo[off] : 0.f);
        if (square) x = x * x;
        t[dy][threadIdx.x] = x;
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t off = b * slab + int64_t(c0 + dy) * R + r0 + threadIdx.x;
        float h, l;
        pair_or_raw(t[threadIdx.x][dy], h, l, dst_lo != nullptr);
        dst_hi[off] = h;
        if (dst_lo) dst_lo[off] = l;
    }
}

void launch_transpose_split(const float* src_hi, const float* src_lo, int nb, int R, int C, float* dst_hi,
                            float* dst_lo, bool square, cudaStream_t s) {
    dim3 grid(C / 32, R / 32, nb), block(32, 8);
    transpose_split_kernel<<<grid, block, 0, s>>>(src_hi, src_lo, R, C, dst_hi, dst_lo, square ? 1 : 0);
    count_launch();
}

// Elementwise (hi + lo)^2, resplit (same layout).
__global__ void square_split_kernel(const float* __restrict__ hi, const float* __restrict__ lo, float* __restrict__ oh,
                                    float* __restrict__ ol, int64_t count) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x) {
        const float x = hi[e] + (lo ? lo[e] : 0.f);
        float h, l;
        pair_or_raw(x * x, h, l, ol != nullptr);
        oh[e] = h;
        if (ol) ol[e] = l;
    }
}

void launch_square_split(const float* hi, const float* lo, float* out_hi, float* out_lo, int64_t count,
                         cudaStream_t s) {
    square_split_kernel<<<1184, 256, 0, s>>>(hi, lo, out_hi, out_lo, count);
    count_launch();
}

// W[b][i][j] = V[b][i][j] * (lam_j + eps_b)^power for j < n (0 beyond), as a
// (hi, lo) split; V is a split [b][D][D] slab. Same clamp / NotPsd rule as
// scale_columns_kernel (densela.hpp:274-278).
__global__ void scale_columns_split_kernel(const float* __restrict__ Vh, const float* __restrict__ Vl,
                                           const double* __restrict__ values, const double* __restrict__ eps,
                                           double power, int n, int D, float* __restrict__ Wh, float* __restrict__ Wl,
                                           int* __restrict__ status) {
    const int64_t b = blockIdx.y;
    const int64_t DD = int64_t(D) * D;
    const double e = eps ? eps[b] : 0.0;
    const double lam_abs = fmax(fabs(values[b * n]), fabs(values[b * n + n - 1]));
    const double tau = 4.0 * 5.9604644775390625e-08 * double(n) * lam_abs;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < DD; idx += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(idx % D);
        float out = 0.f;
        if (j < n) {
            double lam = values[b * n + j];
            if (lam < 0.0 && lam >= -tau) lam = 0.0;
            const double damped = lam + e;
            if (damped <= 0.0) {
                atomicCAS(&status[b], ASG_OK, ASG_ERR_NOT_PSD);
            } else {
                const double v = double(Vh[b * DD + idx]) + (Vl ? double(Vl[b * DD + idx]) : 0.0);
                out = float(v * pow(damped, power));
            }
        }
        float h, l;
        pair_or_raw(out, h, l, Wl != nullptr);
        Wh[b * DD + idx] = h;
        if (Wl) Wl[b * DD + idx] = l;
    }
}

void launch_scale_columns_split(const float* Vh, const float* Vl, const double* values, const double* eps,
                                double power, int nb, int n, int D, float* Wh, float* Wl, int* status,
                                cudaStream_t s) {
    scale_columns_split_kernel<<<dim3(256, nb), 256, 0, s>>>(Vh, Vl, values, eps, power, n, D, Wh, Wl, status);
    count_launch();
}

// eps[b] = damping * tr(A_b) / n from an fp32 [b][M][M] slab.
__global__ void relative_damping_f32_kernel(const float* A, int M, int n, double damping, double* eps) {
    __shared__ double red[32];
    const int64_t b = blockIdx.x;
    double tr = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) tr += double(A[b * int64_t(M) * M + int64_t(i) * M + i]);
    tr = block_reduce_sum(tr, red);
    if (threadIdx.x == 0) eps[b] = n > 0 ? damping * tr / double(n) : 0.0;
}

void launch_relative_damping_f32(const float* A, int nb, int M, int n, double damping, double* eps, cudaStream_t s) {
    relative_damping_f32_kernel<<<nb, 256, 0, s>>>(A, M, n, damping, eps);
    count_launch();
}

// One Newton-Schulz polar step V <- V X, X = (3 I - V^T V) / 2, restores
// orthonormality of an eigenbasis to the fp32 floor (quadratic: 1e-5 -> 1e-10).
// X from S = V^T V (fp32 [b][D][D]) on the leading d x d (zero elsewhere); in
// place of S allowed (Xh == S).
__global__ void ns_x_kernel(const float* S, int d, int D, float* Xh, float* __restrict__ Xl) {
    const int64_t b = blockIdx.y;
    const int64_t DD = int64_t(D) * D;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < DD; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(uint32_t(e) / uint32_t(D)), j = int(uint32_t(e) - uint32_t(i) * uint32_t(D));  // per-matrix index < 2^31
        float x = 0.f;
        if (i < d && j < d) x = (i == j ? 1.5f : 0.f) - 0.5f * S[b * DD + e];
        float h, l;
        pair_or_raw(x, h, l, Xl != nullptr);
        Xh[b * DD + e] = h;
        if (Xl) Xl[b * DD + e] = l;
    }
}

void launch_ns_x(const float* S, int nb, int d, int D, float* Xh, float* Xl, cudaStream_t s) {
    ns_x_kernel<<<dim3(256, nb), 256, 0, s>>>(S, d, D, Xh, Xl);
    count_launch();
}

// out[k] = first failure of (in[k], in[cnt + k]) (both sides of block k).
__global__ void merge_status_kernel(const int* in, int cnt, int* out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    const int a = in[k], b = in[cnt + k];
    if (a != ASG_OK) atomicCAS(&out[k], ASG_OK, a);
    else if (b != ASG_OK) atomicCAS(&out[k], ASG_OK, b);
}

void launch_merge_status(const int* in, int cnt, int* out, cudaStream_t s) {
    merge_status_kernel<<<(cnt + 127) / 128, 128, 0, s>>>(in, cnt, out);
    count_launch();
}

// ============================================================================
// Multi-GPU pack / unpack of block slices (owner-major all-gather layout)
// ============================================================================
// Row-wise: CTA x takes rows x, x + gridDim.x, ...; threads run along the row
// (coalesced on both sides, no per-element index division).
__global__ void pack_kernel(const BlockRef* blocks, const int64_t* offsets, float* out) {
    const BlockRef blk = blocks[blockIdx.y];
    float* o = out + offsets[blockIdx.y];
    for (int r = blockIdx.x; r < blk.rows; r += gridDim.x) {
        const float* src = blk.src + int64_t(r) * blk.ld;
        float* dst = o + int64_t(r) * blk.cols;
        for (int c = threadIdx.x; c < blk.cols; c += blockDim.x) dst[c] = src[c];
    }
}

__global__ void unpack_kernel(const BlockRef* blocks, const int64_t* offsets, const float* in) {
    const BlockRef blk = blocks[blockIdx.y];
    const float* i = in + offsets[blockIdx.y];
    for (int r = blockIdx.x; r < blk.rows; r += gridDim.x) {
        const float* src = i + int64_t(r) * blk.cols;
        float* dst = blk.dst + int64_t(r) * blk.ld;
        for (int c = threadIdx.x; c < blk.cols; c += blockDim.x) dst[c] = src[c];
    }
}

void launch_pack_blocks(const BlockRef* blocks_dev, const int64_t* offsets_dev, int nb, float* out, cudaStream_t s) {
    if (nb > 0) pack_kernel<<<dim3(64, nb), 256, 0, s>>>(blocks_dev, offsets_dev, out);
    count_launch();
}

__global__ void unpack_scaled_kernel(const BlockRef* blocks, const int64_t* offsets, const float* in, float scale) {
    const BlockRef blk = blocks[blockIdx.y];
    const float* i = in + offsets[blockIdx.y];
    for (int r = blockIdx.x; r < blk.rows; r += gridDim.x) {
        const float* src = i + int64_t(r) * blk.cols;
        float* dst = blk.dst + int64_t(r) * blk.ld;
        for (int c = threadIdx.x; c < blk.cols; c += blockDim.x) dst[c] = scale * src[c];
    }
}

void launch_unpack_scaled(const BlockRef* blocks_dev, const int64_t* offsets_dev, int nb, const float* in, float scale,
                          cudaStream_t s) {
    if (nb > 0) unpack_scaled_kernel<<<dim3(64, nb), 256, 0, s>>>(blocks_dev, offsets_dev, in, scale);
    count_launch();
}

void launch_unpack_blocks(const BlockRef* blocks_dev, const int64_t* offsets_dev, int nb, const float* in,
                          cudaStream_t s) {
    if (nb > 0) unpack_kernel<<<dim3(64, nb), 256, 0, s>>>(blocks_dev, offsets_dev, in);
    count_launch();
}


// ============================================================================
// Synthetic gradients: block b at step t is N(0, sigma_b^2)
// i.i.d. from Philox4x32-10 keyed (seed, t, b), one launch for every block.
// Benchmark input generation, not part of the optimizer step.
// ============================================================================
namespace {
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = c.x * 0xD2511F53u, hi0 = __umulhi(c.x, 0xD2511F53u);
        const uint32_t lo1 = c.z * 0xCD9E8D57u, hi1 = __umulhi(c.z, 0xCD9E8D57u);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}
__device__ __forceinline__ float u01(uint32_t x) { return (float(x >> 8) + 0.5f) * (1.0f / 16777216.0f); }  // (0, 1)

// grid (column quads / 256, row groups of kSynthRows, blocks): thread = 4 consecutive
// columns of kSynthRows rows, Philox counter (quad, row, block key) per 4 values; one
// 16-byte store when the row segment is aligned (no per-element index division)
constexpr int kSynthRows = 8;
__global__ void synth_normal_kernel(const SynthBlock* __restrict__ blocks, uint64_t seed, uint64_t step) {
    const SynthBlock b = blocks[blockIdx.z];
    const int q = blockIdx.x * blockDim.x + threadIdx.x;  // column quad
    if (4 * q >= b.cols) return;
    const uint2 key = make_uint2(uint32_t(seed) ^ uint32_t(step * 0x9E3779B97F4A7C15ull),
                                 uint32_t(seed >> 32) ^ uint32_t((step * 0x9E3779B97F4A7C15ull) >> 32));
    const int row1 = min(b.rows, int(blockIdx.y + 1) * kSynthRows);
#pragma unroll 2
    for (int row = blockIdx.y * kSynthRows; row < row1; ++row) {
    const uint4 r = philox4x32_10(make_uint4(uint32_t(q), uint32_t(row), b.key, 0u), key);
    const float r1 = sqrtf(-2.f * __logf(u01(r.x))), r2 = sqrtf(-2.f * __logf(u01(r.z)));
    float s1, c1, s2, c2;
    __sincosf(6.2831853f * u01(r.y), &s1, &c1);
    __sincosf(6.2831853f * u01(r.w), &s2, &c2);
    const float4 z = make_float4(b.sigma * r1 * c1, b.sigma * r1 * s1, b.sigma * r2 * c2, b.sigma * r2 * s2);
    float* d = b.dst + int64_t(row) * b.ld + 4 * q;
    if (4 * q + 3 < b.cols && (reinterpret_cast<uintptr_t>(d) & 15) == 0) {
        *reinterpret_cast<float4*>(d) = z;
    } else {
        const float zz[4] = {z.x, z.y, z.z, z.w};
        for (int j = 0; j < 4 && 4 * q + j < b.cols; ++j) d[j] = zz[j];
    }
    }
}
}  // namespace

void launch_synth_normal(const SynthBlock* blocks_dev, int nb, int max_rows, int max_cols, uint64_t seed,
                         uint64_t step, cudaStream_t s) {
    if (nb <= 0 || max_rows <= 0 || max_cols <= 0) return;
    const int quads = (max_cols + 3) / 4;
    synth_normal_kernel<<<dim3((quads + 255) / 256, (max_rows + kSynthRows - 1) / kSynthRows, nb), 256, 0, s>>>(
        blocks_dev, seed, step);
    count_launch();
}


// ============================================================================
// 3xFP16 operands: power-of-two scales and (hi, lo) fp16 pairs
// ============================================================================
namespace {
// s = 2^(14 - floor(log2 m)): m s in [2^14, 2^15) (max fp16 65504); 1 for m == 0 / non-finite
__device__ __forceinline__ float f16_scale(unsigned int mbits) {
    const int e = int((mbits >> 23) & 0xff);
    if (e == 0 || e == 0xff) return 1.f;
    const int ex = 268 - e;  // biased exponent of 2^(14 - (e - 127))
    return __uint_as_float(uint32_t(ex > 254 ? 254 : ex) << 23);
}
__device__ __forceinline__ void f16_split(float y, __half& h, __half& l) {
    h = __float2half_rn(y);
    l = __float2half_rn(y - __half2float(h));
}

__device__ __forceinline__ float absmax4(const float4 v) {
    const float m = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
    return isfinite(v.x + v.y + v.z + v.w) ? m : __int_as_float(0x7f800000);
}
// one atomic per CTA (256 threads)
__device__ __forceinline__ void block_max_atomic(float m, unsigned int* dst) {
    __shared__ float red[8];
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
        atomicMax(dst, __float_as_uint(m));
    }
}

__global__ void __launch_bounds__(256) absmax_kernel(const float* __restrict__ src, int64_t per,
                                                     unsigned int* __restrict__ amax) {
    const int64_t b = blockIdx.y;
    const float4* p4 = reinterpret_cast<const float4*>(src + b * per);
    const int64_t n4 = per / 4, stride = int64_t(gridDim.x) * blockDim.x;
    float m = 0.f;
    int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {  // four loads in flight per thread
        const float4 v0 = p4[i], v1 = p4[i + stride], v2 = p4[i + 2 * stride], v3 = p4[i + 3 * stride];
        m = fmaxf(m, fmaxf(fmaxf(absmax4(v0), absmax4(v1)), fmaxf(absmax4(v2), absmax4(v3))));
    }
    for (; i < n4; i += stride) m = fmaxf(m, absmax4(p4[i]));
    block_max_atomic(m, amax + b);
}

__global__ void to_f16pair_kernel(const float* __restrict__ src, const unsigned int* __restrict__ amax, int64_t per,
                                  __half* __restrict__ hi, __half* __restrict__ lo, float* __restrict__ scale) {
    const int64_t b = blockIdx.y;
    const float s = f16_scale(amax[b]);
    if (blockIdx.x == 0 && threadIdx.x == 0) scale[b] = s;
    const float4* p4 = reinterpret_cast<const float4*>(src + b * per);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < per / 4; i += int64_t(gridDim.x) * blockDim.x) {
        const float4 v = p4[i];
        __half h[4], l[4];
        f16_split(v.x * s, h[0], l[0]);
        f16_split(v.y * s, h[1], l[1]);
        f16_split(v.z * s, h[2], l[2]);
        f16_split(v.w * s, h[3], l[3]);
        *reinterpret_cast<uint2*>(hi + b * per + 4 * i) = *reinterpret_cast<const uint2*>(h);
        *reinterpret_cast<uint2*>(lo + b * per + 4 * i) = *reinterpret_cast<const uint2*>(l);
    }
}

// max over columns of sum_i |P_ij| (the 1-norm) of each n x n slot, as float bits.
// 32 x 32 threads per 32-column strip: warp y sums rows y, y+32, ... (one 128-byte row
// segment per load), the 32 partial sums of a column are combined in shared memory.
__global__ void __launch_bounds__(1024) colabs_max_kernel(const float* __restrict__ src, int n, int64_t per,
                                                          unsigned int* __restrict__ out) {
    __shared__ float part[32][33];
    const int j = blockIdx.x * 32 + threadIdx.x;
    const float* p = src + int64_t(blockIdx.y) * per;
    float a0 = 0.f, a1 = 0.f;
    if (j < n) {
        int i = threadIdx.y;
        for (; i + 32 < n; i += 64) {
            a0 += fabsf(p[int64_t(i) * n + j]);
            a1 += fabsf(p[int64_t(i + 32) * n + j]);
        }
        if (i < n) a0 += fabsf(p[int64_t(i) * n + j]);
    }
    part[threadIdx.y][threadIdx.x] = a0 + a1;
    __syncthreads();
    if (threadIdx.y == 0) {
        float c = 0.f;
        for (int y = 0; y < 32; ++y) c += part[y][threadIdx.x];
        if (!isfinite(c)) c = __int_as_float(0x7f800000);
        for (int o = 16; o > 0; o >>= 1) c = fmaxf(c, __shfl_xor_sync(0xffffffffu, c, o));
        if (threadIdx.x == 0) atomicMax(out + blockIdx.y, __float_as_uint(c));
    }
}

// the fp16 output scale of D = A B with |D_ij| <= max|A| ||B||_1: max|A| < 2^15 / ascale (the
// fp16 scale of A puts max|A| ascale in [2^14, 2^15)), so D's bound is 2^15 ||B||_1 / ascale
__global__ void bound_scale_kernel(int nb, const float* __restrict__ ascale, const unsigned int* __restrict__ n1,
                                   float* __restrict__ out0, float* __restrict__ out1) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const float bound = 32768.f / ascale[b] * __uint_as_float(n1[b]);
    const float s = f16_scale(__float_as_uint(bound));
    out0[b] = s;
    if (out1) out1[b] = s;
}

// max |x| over each gradient block's view (rows x cols of the caller's tensor)
__global__ void block_absmax_kernel(const BlockRef* __restrict__ blocks, unsigned int* __restrict__ amax) {
    const BlockRef blk = blocks[blockIdx.y];
    float m = 0.f;
    for (int i = blockIdx.x; i < blk.rows; i += gridDim.x)
        for (int j = threadIdx.x; j < blk.cols; j += blockDim.x) {
            const float x = blk.src[int64_t(i) * blk.ld + j];
            m = isfinite(x) ? fmaxf(m, fabsf(x)) : __int_as_float(0x7f800000);
        }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(amax + blockIdx.y, __float_as_uint(m));
}

// G (x scale_val, x the block's fp16 scale) -> fp16 pairs of G [b][M][N] and G^T [b][N][M]
__global__ void prep_grad_f16_kernel(const BlockRef* __restrict__ blocks, int M, int N, float scale_val,
                                     const unsigned int* __restrict__ amax, __half* __restrict__ Gh,
                                     __half* __restrict__ Gl, __half* __restrict__ GTh, __half* __restrict__ GTl,
                                     float* __restrict__ gscale) {
    __shared__ float t[32][33];
    const int b = blockIdx.z;
    const BlockRef blk = blocks[b];
    // the scale covers the clip-scaled values: max |scale_val x| = scale_val max |x|
    const float s = f16_scale(__float_as_uint(__uint_as_float(amax[b]) * scale_val));
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0) gscale[b] = s;
    const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    const int64_t slab = int64_t(M) * N;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int i = i0 + dy, j = j0 + threadIdx.x;
        float x = 0.f;
        if (i < blk.rows && j < blk.cols) x = scale_val * blk.src[int64_t(i) * blk.ld + j] * s;
        __half h, l;
        f16_split(x, h, l);
        Gh[b * slab + int64_t(i) * N + j] = h;
        Gl[b * slab + int64_t(i) * N + j] = l;
        t[dy][threadIdx.x] = x;
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int jj = j0 + dy, ii = i0 + threadIdx.x;
        __half h, l;
        f16_split(t[threadIdx.x][dy], h, l);
        GTh[b * slab + int64_t(jj) * M + ii] = h;
        GTl[b * slab + int64_t(jj) * M + ii] = l;
    }
}
// float4 variants for blocks whose rows are 16-byte aligned (BlockRef src, ld, cols % 4 == 0)
// (rows x cols/4) float4 cells of the block flattened, four loads in flight per thread
__global__ void __launch_bounds__(256) block_absmax_vec_kernel(const BlockRef* __restrict__ blocks,
                                                               unsigned int* __restrict__ amax) {
    const BlockRef blk = blocks[blockIdx.y];
    const int c4 = blk.cols / 4;
    const int64_t n4 = int64_t(blk.rows) * c4, stride = int64_t(gridDim.x) * blockDim.x;
    auto at = [&](int64_t q) {
        const int64_t r = q / c4;
        return *reinterpret_cast<const float4*>(blk.src + r * blk.ld + 4 * (q - r * c4));
    };
    float m = 0.f;
    int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    for (; q + 3 * stride < n4; q += 4 * stride) {
        const float4 v0 = at(q), v1 = at(q + stride), v2 = at(q + 2 * stride), v3 = at(q + 3 * stride);
        m = fmaxf(m, fmaxf(fmaxf(absmax4(v0), absmax4(v1)), fmaxf(absmax4(v2), absmax4(v3))));
    }
    for (; q < n4; q += stride) m = fmaxf(m, absmax4(at(q)));
    block_max_atomic(m, amax + blockIdx.y);
}

// 64 x 64 tiles, 16 x 16 threads: float4 loads, 8-byte fp16 stores of 4 (hi, lo) values per row segment
__global__ void __launch_bounds__(256) prep_grad_f16_vec_kernel(const BlockRef* __restrict__ blocks, int M, int N,
                                                                float scale_val, const unsigned int* __restrict__ amax,
                                                                __half* __restrict__ Gh, __half* __restrict__ Gl,
                                                                __half* __restrict__ GTh, __half* __restrict__ GTl,
                                                                float* __restrict__ gscale) {
    __shared__ float t[64][65];
    const int b = blockIdx.z;
    const BlockRef blk = blocks[b];
    const float s = f16_scale(__float_as_uint(__uint_as_float(amax[b]) * scale_val));
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0) gscale[b] = s;
    const float f = scale_val * s;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int j0 = blockIdx.x * 64, i0 = blockIdx.y * 64;
    const int64_t slab = int64_t(M) * N;
    auto put4 = [](__half* hp, __half* lp, float a, float bb, float c, float d) {
        __half h[4], l[4];
        f16_split(a, h[0], l[0]);
        f16_split(bb, h[1], l[1]);
        f16_split(c, h[2], l[2]);
        f16_split(d, h[3], l[3]);
        *reinterpret_cast<uint2*>(hp) = *reinterpret_cast<const uint2*>(h);
        *reinterpret_cast<uint2*>(lp) = *reinterpret_cast<const uint2*>(l);
    };
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int i = i0 + ty + 16 * r, j = j0 + tx * 4;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < blk.rows && j < blk.cols) x = *reinterpret_cast<const float4*>(blk.src + int64_t(i) * blk.ld + j);
        x = make_float4(f * x.x, f * x.y, f * x.z, f * x.w);
        const int64_t o = b * slab + int64_t(i) * N + j;
        put4(Gh + o, Gl + o, x.x, x.y, x.z, x.w);
        const int rr = ty + 16 * r, cc = tx * 4;
        t[rr][cc] = x.x;
        t[rr][cc + 1] = x.y;
        t[rr][cc + 2] = x.z;
        t[rr][cc + 3] = x.w;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int jj = j0 + ty + 16 * r, ii = i0 + tx * 4;  // GT[jj][ii..ii+3] = G[ii..ii+3][jj]
        const int cc = ty + 16 * r, rr = tx * 4;
        const int64_t o = b * slab + int64_t(jj) * M + ii;
        put4(GTh + o, GTl + o, t[rr][cc], t[rr + 1][cc], t[rr + 2][cc], t[rr + 3][cc]);
    }
}

// 3xFP16 gradient prep without a separate max pass: G and G^T are written at the scale
// predicted from the previous step's max of the same block (pred, raw |G| bits; two binades
// of headroom), while this step's max is accumulated into `now`. prep_f16_check_kernel then
// flags the blocks whose prediction was unsafe (overflow risk) or too loose (< 2^2 of fp16's
// top binade used) -- and every block on the first step (pred = 0) -- and the same kernel in
// FIX mode (fix != nullptr) rewrites just those blocks at the exact scale of `now`. The main
// pass runs one 64 x 64 tile per CTA; the FIX pass is grid-stride over (block, tile) and
// returns at once when no block is flagged (one load per thread).
__global__ void __launch_bounds__(256) prep_grad_f16_pred_kernel(const BlockRef* __restrict__ blocks, int nb, int M,
                                                                 int N, float scale_val,
                                                                 const unsigned int* __restrict__ pred,
                                                                 unsigned int* __restrict__ now,
                                                                 const int* __restrict__ fix, __half* __restrict__ Gh,
                                                                 __half* __restrict__ Gl, __half* __restrict__ GTh,
                                                                 __half* __restrict__ GTl, float* __restrict__ gscale) {
    __shared__ float t[64][65];
    __shared__ float red[8];
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 16 + tx;
    const int tj = N / 64, ti = M / 64, per = ti * tj;
    const int64_t slab = int64_t(M) * N;
    auto put4 = [](__half* hp, __half* lp, float a, float bb, float c, float d) {
        __half h[4], l[4];
        f16_split(a, h[0], l[0]);
        f16_split(bb, h[1], l[1]);
        f16_split(c, h[2], l[2]);
        f16_split(d, h[3], l[3]);
        *reinterpret_cast<uint2*>(hp) = *reinterpret_cast<const uint2*>(h);
        *reinterpret_cast<uint2*>(lp) = *reinterpret_cast<const uint2*>(l);
    };
    if (fix) {
        int any = 0;
        for (int b = tid; b < nb; b += 256) any |= fix[b];
        if (!__syncthreads_or(any)) return;
    }
    const int64_t w0 = fix ? blockIdx.x : (int64_t(blockIdx.z) * ti + blockIdx.y) * tj + blockIdx.x;
    const int64_t wstep = fix ? gridDim.x : int64_t(nb) * per;
    for (int64_t w = w0; w < int64_t(nb) * per; w += wstep) {
        const int b = int(w / per), tile = int(w - int64_t(b) * per);
        if (fix && !fix[b]) continue;  // block-uniform
        const BlockRef blk = blocks[b];
        const float s = fix ? f16_scale(__float_as_uint(__uint_as_float(now[b]) * scale_val))
                            : (pred[b] ? f16_scale(__float_as_uint(__uint_as_float(pred[b]) * scale_val * 4.f)) : 1.f);
        if (tile == 0 && tid == 0) gscale[b] = s;
        const float f = scale_val * s;
        const int j0 = (tile % tj) * 64, i0 = (tile / tj) * 64;
        float mx = 0.f;
        float4 xs[4];  // all four loads in flight before the first store
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = i0 + ty + 16 * r, j = j0 + tx * 4;
            xs[r] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (i < blk.rows && j < blk.cols) xs[r] = __ldcs(reinterpret_cast<const float4*>(blk.src + int64_t(i) * blk.ld + j));
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = i0 + ty + 16 * r, j = j0 + tx * 4;
            float4 x = xs[r];
            mx = fmaxf(mx, absmax4(x));
            x = make_float4(f * x.x, f * x.y, f * x.z, f * x.w);
            const int64_t o = b * slab + int64_t(i) * N + j;
            put4(Gh + o, Gl + o, x.x, x.y, x.z, x.w);
            const int rr = ty + 16 * r, cc = tx * 4;
            t[rr][cc] = x.x;
            t[rr][cc + 1] = x.y;
            t[rr][cc + 2] = x.z;
            t[rr][cc + 3] = x.w;
        }
        if (!fix) {  // this step's max |G| of the block (raw)
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if ((tid & 31) == 0) red[tid >> 5] = mx;
        }
        __syncthreads();
        if (!fix && tid == 0) {
            for (int k = 1; k < 8; ++k) mx = fmaxf(mx, red[k]);
            atomicMax(now + b, __float_as_uint(mx));
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int jj = j0 + ty + 16 * r, ii = i0 + tx * 4;  // GT[jj][ii..ii+3] = G[ii..ii+3][jj]
            const int cc = ty + 16 * r, rr = tx * 4;
            const int64_t o = b * slab + int64_t(jj) * M + ii;
            put4(GTh + o, GTl + o, t[rr][cc], t[rr + 1][cc], t[rr + 2][cc], t[rr + 3][cc]);
        }
        __syncthreads();
    }
}

__global__ void prep_f16_check_kernel(int nb, float scale_val, unsigned int* __restrict__ pred,
                                      const unsigned int* __restrict__ now, const float* __restrict__ gscale,
                                      int* __restrict__ fix) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const float m = __uint_as_float(now[b]) * scale_val, y = m * gscale[b];
    fix[b] = (m == 0.f || (y >= 4.f && y < 32768.f)) ? 0 : 1;  // (non-finite: fixed, then reported downstream)
    pred[b] = now[b];
}
}  // namespace

void launch_prep_grad_f16_pred(const BlockRef* blocks_dev, int nb, int M, int N, float scale_val, unsigned int* pred,
                               unsigned int* now, int* fix, void* Gh16, void* Gl16, void* GTh16, void* GTl16,
                               float* gscale, cudaStream_t s) {
    if (nb <= 0) return;
    cudaMemsetAsync(now, 0, size_t(nb) * sizeof(unsigned int), s);
    const int64_t work = int64_t(nb) * (M / 64) * (N / 64);
    const int grid = int(std::min<int64_t>(work, 148 * 8));
    auto* gh = static_cast<__half*>(Gh16);
    auto* gl = static_cast<__half*>(Gl16);
    auto* th = static_cast<__half*>(GTh16);
    auto* tl = static_cast<__half*>(GTl16);
    prep_grad_f16_pred_kernel<<<dim3(N / 64, M / 64, nb), dim3(16, 16), 0, s>>>(blocks_dev, nb, M, N, scale_val, pred,
                                                                                now, nullptr, gh, gl, th, tl, gscale);
    prep_f16_check_kernel<<<(nb + 127) / 128, 128, 0, s>>>(nb, scale_val, pred, now, gscale, fix);
    prep_grad_f16_pred_kernel<<<grid, dim3(16, 16), 0, s>>>(blocks_dev, nb, M, N, scale_val, pred, now, fix, gh, gl, th,
                                                            tl, gscale);
    count_launch(3);
}

void launch_colabs_max(const float* src, int nb, int n, int64_t per, unsigned int* out, cudaStream_t s) {
    if (nb <= 0) return;
    cudaMemsetAsync(out, 0, size_t(nb) * sizeof(unsigned int), s);
    colabs_max_kernel<<<dim3((n + 31) / 32, nb), dim3(32, 32), 0, s>>>(src, n, per, out);
    count_launch(1);
}

void launch_bound_scale(int nb, const float* ascale, const unsigned int* n1, float* out0, float* out1, cudaStream_t s) {
    if (nb <= 0) return;
    bound_scale_kernel<<<(nb + 127) / 128, 128, 0, s>>>(nb, ascale, n1, out0, out1);
    count_launch(1);
}

void launch_absmax(const float* src, int nb, int64_t per, unsigned int* amax, cudaStream_t s) {
    if (nb <= 0) return;
    cudaMemsetAsync(amax, 0, size_t(nb) * sizeof(unsigned int), s);
    // about 8 CTAs per SM over the whole batch, each thread with >= 16 float4 of work
    const int64_t want = (8 * 148 + nb - 1) / nb;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(want, (per / 4 + 4095) / 4096));
    absmax_kernel<<<dim3(unsigned(blocks > 0 ? blocks : 1), nb), 256, 0, s>>>(src, per, amax);
    count_launch();
}

void launch_to_f16pair(const float* src, const unsigned int* amax, int nb, int64_t per, void* hi16, void* lo16,
                       float* scale, cudaStream_t s) {
    if (nb <= 0) return;
    const int64_t blocks = std::min<int64_t>(1024, (per / 4 + 255) / 256);
    to_f16pair_kernel<<<dim3(unsigned(blocks > 0 ? blocks : 1), nb), 256, 0, s>>>(
        src, amax, per, static_cast<__half*>(hi16), static_cast<__half*>(lo16), scale);
    count_launch();
}

void launch_prep_grad_f16(const BlockRef* blocks_dev, int nb, int M, int N, float scale_val, unsigned int* amax,
                          void* Gh16, void* Gl16, void* GTh16, void* GTl16, float* gscale, cudaStream_t s, bool vec) {
    if (nb <= 0) return;
    cudaMemsetAsync(amax, 0, size_t(nb) * sizeof(unsigned int), s);
    if (vec && M % 64 == 0 && N % 64 == 0) {
        const int want = (8 * 148 + nb - 1) / nb;
        const int gx = std::max(1, std::min(want, int((int64_t(M) * N / 4 + 4095) / 4096)));
        block_absmax_vec_kernel<<<dim3(gx, nb), 256, 0, s>>>(blocks_dev, amax);
        prep_grad_f16_vec_kernel<<<dim3(N / 64, M / 64, nb), dim3(16, 16), 0, s>>>(
            blocks_dev, M, N, scale_val, amax, static_cast<__half*>(Gh16), static_cast<__half*>(Gl16),
            static_cast<__half*>(GTh16), static_cast<__half*>(GTl16), gscale);
    } else {
        block_absmax_kernel<<<dim3(std::min(M, 256), nb), 256, 0, s>>>(blocks_dev, amax);
        prep_grad_f16_kernel<<<dim3(N / 32, M / 32, nb), dim3(32, 8), 0, s>>>(
            blocks_dev, M, N, scale_val, amax, static_cast<__half*>(Gh16), static_cast<__half*>(Gl16),
            static_cast<__half*>(GTh16), static_cast<__half*>(GTl16), gscale);
    }
    count_launch(2);
}

}  // namespace asg
