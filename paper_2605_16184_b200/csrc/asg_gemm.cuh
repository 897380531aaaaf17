// SPDX-License-Identifier: Apache-2.0
//
// Batched "TN" tensor-core GEMM for sm_100a with fused optimizer epilogues.
//
//   acc[b] = A[b] * B[b]^T        A: [batch][M][K] fp32, B: [batch][N][K] fp32
//
// Both operands are K-major (row-major with K contiguous), staged by TMA into
// 128B-swizzled shared memory, multiplied by tcgen05.mma kind::tf32 into an
// fp32 accumulator in TMEM, and drained by eight epilogue warps with
// tcgen05.ld. Precision: NPASS=1 is plain TF32; NPASS=3 is 3xTF32, where every
// operand is given as an exact (hi, lo) tf32 pair and the kernel accumulates
// hi*hi + hi*lo + lo*hi — fp32-faithful products (relative error ~2^-21).
//
// Persistent: one CTA per SM loops over output tiles (128 x BN). Warp roles:
//   warp 0: TMA producer      warp 1: MMA issuer + TMEM owner
//   warps 2-9: epilogue (TMEM lane quadrant = warp % 4; the two warps of a
//              quadrant split the tile's 32-column chunks, doubling the
//              memory parallelism of the fused epilogues)
// Pipelines: smem stages full/empty (TMA <-> MMA) and a double-buffered TMEM
// accumulator tfull/tempty (MMA <-> epilogue), so tile t's epilogue overlaps
// tile t+1's MMAs.
//
// Epilogues (the reference op each one fuses is cited):
//   EPI_STORE    C = alpha*acc + beta*C                        (diagnostics)
//   EPI_SYM_EMA  C = beta*C + alpha*acc on the lower triangle, mirrored to the
//                upper (accumulate_factors precond.cpp:181-188 incl. the
//                symmetrize of densela.hpp:152-156: C stays exactly symmetric)
//   EPI_SPLIT    D = alpha*acc written as a (hi, lo) tf32 pair (next GEMM's A)
//   EPI_SPLIT_T  same, transposed (next GEMM's B)
//   EPI_ADAM     Adam in the rotated basis (soap_scaled_step precond.cpp:213-221):
//                updates m, v in place, writes S = m^/(sqrt(v^)+eps) as (hi, lo)
//   EPI_APPLY    theta -= lr*lr_scale*(alpha*acc + wd*theta) on the block's
//                slice of the caller's parameter (apply_update precond.cpp:244-251)
//   EPI_SYM_SPLIT  D = alpha*acc as a (hi, lo) pair on the lower triangle,
//                mirrored (products of commuting symmetric matrices: the
//                coupled Newton-Schulz inverse root, asg_newton.cu)
//   EPI_NS       EPI_SYM_SPLIT for M, plus T = ns_a*I - ns_b*M as a second
//                (hi, lo) pair and max|M - I| per batch into resid[b]
//   EPI_SPLIT2   EPI_SPLIT, plus the transpose as a second (hi, lo) pair in
//                Thi/Tlo (leading dimension ldt): both operand layouts of one
//                product (KL-Shampoo's V^T = G^T P_L, asg_runtime.cu group_stats)
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "asg_ptx.cuh"

namespace asg {

enum EpiKind {
    EPI_STORE = 0,
    EPI_SYM_EMA = 1,
    EPI_SPLIT = 2,
    EPI_SPLIT_T = 3,
    EPI_ADAM = 4,
    EPI_APPLY = 5,
    EPI_SYM_SPLIT = 6,
    EPI_NS = 7,
    EPI_SPLIT2 = 8
};

struct ApplyEntry {
    float* theta;   // first element of the block inside the parameter
    int64_t ld;     // parameter leading dimension
    int32_t rows;   // block extent (unpadded)
    int32_t cols;
};

struct GemmParams {
    int M, N, K, batch;   // padded per-batch problem
    int tiles_n;          // N / BN
    int tiles_per_batch;  // rectangular: (M/128)*(N/BN); symmetric: list length
    int num_tiles;        // batch * tiles_per_batch
    const int2* tile_list;  // symmetric schedules: (tile_m, tile_n) per batch-local tile
    float alpha, beta;
    float* C;             // EPI_STORE / EPI_SYM_EMA output
    int64_t ldc, c_bstride;
    float* Dhi;           // EPI_SPLIT / EPI_SPLIT_T / EPI_ADAM outputs
    float* Dlo;
    int64_t ldd, d_bstride;
    float* mom_m;         // EPI_ADAM moments, [batch][M][N]
    float* mom_v;
    int64_t ldm, m_bstride;
    float b1, b2, inv_bc1, inv_bc2, adam_eps;
    const ApplyEntry* apply;  // EPI_APPLY: per batch entry
    float lr_eff, wd;
    int* flag;            // set to 1 on a non-finite update (EPI_APPLY)
    const int* batch_active;  // optional: batches with batch_active[b] == 0 are skipped (no output)
    float* Thi;           // EPI_NS: T = ns_a I - ns_b M (hi, lo), same layout as D; EPI_SPLIT2: D^T
    float* Tlo;
    int64_t ldt;          // EPI_SPLIT2: leading dimension of D^T (batch stride d_bstride)
    float ns_a, ns_b;
    unsigned int* resid;  // EPI_NS: per batch max|M - I| (float bits, atomicMax)
    int raster;           // rectangular schedules: 0 row-major tiles, 1 column-major
    int raw_out;          // 3xTF32: an output without a lo array stores the full fp32 value
    int a_raw, b_raw;     // SPL kernels: operand given as plain fp32 (split in shared memory)
    const float* ascale;  // F16 kernels: per-batch power-of-two scales the fp16 operands carry
    const float* bscale;  //   (the accumulator is divided by ascale[b] * bscale[b])
    unsigned int* omax;   // optional: per-batch max |output| (float bits, atomicMax) of SPLIT / SPLIT2
    int sym_T;            // CTA-pair symmetric schedules: T x T tile grid, lower triangle decoded
                          // arithmetically (tile_list unused)
    const float* oscale;  // SPLIT / SPLIT2 / SYM_SPLIT / NS fp16-pair output: D (and D^T, T) are written
                          // as scaled fp16 (hi, lo) pairs, __half arrays at Dhi/Dlo (Thi/Tlo), value * oscale[b]
};

__device__ __forceinline__ bool batch_skipped(const GemmParams& p, int t) {
    return p.batch_active && p.batch_active[t / p.tiles_per_batch] == 0;
}

// An output operand value: a (hi, lo) tf32 pair when the lo array exists;
// otherwise the full fp32 value in 3xTF32 mode (its consumer splits it in
// shared memory, gemm_tn_kernel<..., SPL>) or its tf32 rounding in TF32 mode.
__device__ __forceinline__ void out_split(const GemmParams& p, float x, float& hi, float& lo, bool has_lo) {
    if (has_lo)
        split_tf32(x, hi, lo);
    else
        hi = p.raw_out ? x : tf32_round(x);
}

// CG = 1: one CTA per 128 x BN tile. CG = 2: a CTA pair (cluster (2,1,1),
// tcgen05 cta_group::2) per 256 x BN tile; each CTA stages 128 rows of A and
// BN/2 rows of B, so the per-SM operand bytes (shared-memory reads of the
// MMA, TMA writes) drop by a third at BN = 256 and the ring gets deeper.
// SPL (3xTF32 only): operands flagged raw (GemmParams::a_raw / b_raw) arrive
// as plain fp32; four converter warps write each staged tile's lo part in
// shared memory (the stage keeps its (hi, lo) layout; either operand may be
// raw), so HBM holds and streams one fp32 per element. (A variant with a
// deeper hi-only TMA ring and a separate 2-slot lo ring measured 1.4x slower
// per launch: the conversion, not the load latency, sets the pace.)
// F16: 3xFP16 -- every operand is an exact (hi, lo) pair of fp16 values
// carrying a per-matrix power-of-two scale (x * s = hi + lo to ~2^-22;
// max |x| s in [2^14, 2^15)), multiplied by tcgen05.mma kind::f16 at twice the
// tf32 rate per staged byte; a 128-byte smem row then holds 64 K elements.
template <int BN, int NPASS, int CG = 1, bool SPL = false, bool F16 = false>
struct GemmCfg {
    static constexpr int BM = 128;       // accumulator rows per CTA
    static constexpr int TM = 128 * CG;  // output tile rows
    static constexpr int BK = F16 ? 64 : 32;  // K elements per 128-byte swizzle row
    static constexpr bool kSplit = NPASS > 1;
    static constexpr int kBRows = BN / CG;  // B rows staged by each CTA
    static constexpr uint32_t kABytes = BM * 128;
    static constexpr uint32_t kBBytes = kBRows * 128;
    static constexpr uint32_t kStageBytes = (kABytes + kBBytes) * (kSplit ? 2 : 1);
    // per-epilogue-warp 32 x 33 fp32 transpose scratch (coalesced apply)
    static constexpr int kEpiWarps = 8;
    static constexpr int kConvWarps = SPL ? 4 : 0;  // warps 2 + kEpiWarps ...
    static_assert(SPL == 0 || ((kABytes / 16) % 512 == 0 && (kBBytes / 16) % 512 == 0),
                  "converter: whole 4 x 128-thread batches of 16-byte words");
    static constexpr int kThreads = 32 * (2 + kEpiWarps + kConvWarps);
    static constexpr uint32_t kScratchBytes = kEpiWarps * 32 * 33 * 4;
    static constexpr int kStagesRaw = int((194 * 1024) / kStageBytes);
    static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
    static constexpr size_t kRingBytes = size_t(kStages) * kStageBytes;
    static constexpr uint32_t kTmemCols = 2 * BN;  // double-buffered accumulator
    static constexpr size_t kSmemBytes = 1024 /*align slack*/ + kRingBytes + 256 + kScratchBytes;
    static_assert(kStages >= 2, "need at least two pipeline stages");
    static_assert(kTmemCols == 256 || kTmemCols == 512, "TMEM allocation must be a power of two");
};

__device__ __forceinline__ void decode_tile(const GemmParams& p, int t, int& b, int& tm, int& tn) {
    b = t / p.tiles_per_batch;
    const int l = t - b * p.tiles_per_batch;
    if (p.sym_T) {  // lower triangle of a T x T grid, row by row: l = tm (tm + 1) / 2 + tn
        int r = int((sqrtf(8.f * float(l) + 1.f) - 1.f) * 0.5f);
        while (r * (r + 1) / 2 > l) --r;
        while ((r + 1) * (r + 2) / 2 <= l) ++r;
        tm = r;
        tn = l - r * (r + 1) / 2;
    } else if (p.tile_list) {
        const int2 c = p.tile_list[l];
        tm = c.x;
        tn = c.y;
    } else {
        if (p.raster == 1) {  // column-major: consecutive tiles share the B panel
            const int tiles_m = p.tiles_per_batch / p.tiles_n;
            tn = l / tiles_m;
            tm = l - tn * tiles_m;
        } else {
            tm = l / p.tiles_n;
            tn = l - tm * p.tiles_n;
        }
    }
}

// One thread owns one accumulator row (`row`) and 32 consecutive columns.
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int b, int row, int col0,
                                               const uint32_t (&r)[32]) {
    if constexpr (EPI == EPI_STORE) {
        float* c = p.C + int64_t(b) * p.c_bstride + int64_t(row) * p.ldc + col0;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            float4 v;
            v.x = p.alpha * __uint_as_float(r[j + 0]);
            v.y = p.alpha * __uint_as_float(r[j + 1]);
            v.z = p.alpha * __uint_as_float(r[j + 2]);
            v.w = p.alpha * __uint_as_float(r[j + 3]);
            if (p.beta != 0.f) {
                const float4 o = *reinterpret_cast<const float4*>(c + j);
                v.x += p.beta * o.x;
                v.y += p.beta * o.y;
                v.z += p.beta * o.z;
                v.w += p.beta * o.w;
            }
            *reinterpret_cast<float4*>(c + j) = v;
        }
    } else if constexpr (EPI == EPI_SYM_EMA) {
        float* cb = p.C + int64_t(b) * p.c_bstride;
        if (row < col0) return;  // whole chunk strictly above the diagonal
        float* crow = cb + int64_t(row) * p.ldc + col0;
        float vals[32];
        if (p.beta != 0.f) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const float4 o = *reinterpret_cast<const float4*>(crow + j);
                vals[j + 0] = p.beta * o.x + p.alpha * __uint_as_float(r[j + 0]);
                vals[j + 1] = p.beta * o.y + p.alpha * __uint_as_float(r[j + 1]);
                vals[j + 2] = p.beta * o.z + p.alpha * __uint_as_float(r[j + 2]);
                vals[j + 3] = p.beta * o.w + p.alpha * __uint_as_float(r[j + 3]);
            }
        } else {  // C need not be initialised (scratch)
#pragma unroll
            for (int j = 0; j < 32; ++j) vals[j] = p.alpha * __uint_as_float(r[j]);
        }
        if (row >= col0 + 31) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(crow + j) = make_float4(vals[j], vals[j + 1], vals[j + 2], vals[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (row >= col0 + j) crow[j] = vals[j];
        }
        // Mirror: C[c][row] for c < row; consecutive lanes hit consecutive rows' column.
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (row > col0 + j) cb[int64_t(col0 + j) * p.ldc + row] = vals[j];
    } else if constexpr (EPI == EPI_SPLIT) {
        const int64_t off = int64_t(b) * p.d_bstride + int64_t(row) * p.ldd + col0;
        float* dh = p.Dhi + off;
        float* dl = p.Dlo + off;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            float4 h, l;
            out_split(p, p.alpha * __uint_as_float(r[j + 0]), h.x, l.x, p.Dlo != nullptr);
            out_split(p, p.alpha * __uint_as_float(r[j + 1]), h.y, l.y, p.Dlo != nullptr);
            out_split(p, p.alpha * __uint_as_float(r[j + 2]), h.z, l.z, p.Dlo != nullptr);
            out_split(p, p.alpha * __uint_as_float(r[j + 3]), h.w, l.w, p.Dlo != nullptr);
            *reinterpret_cast<float4*>(dh + j) = h;
            if (p.Dlo) *reinterpret_cast<float4*>(dl + j) = l;
        }
    } else if constexpr (EPI == EPI_SPLIT_T) {
        float* dh = p.Dhi + int64_t(b) * p.d_bstride + row;
        float* dl = p.Dlo + int64_t(b) * p.d_bstride + row;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            float h, l;
            out_split(p, p.alpha * __uint_as_float(r[j]), h, l, p.Dlo != nullptr);
            dh[int64_t(col0 + j) * p.ldd] = h;
            if (p.Dlo) dl[int64_t(col0 + j) * p.ldd] = l;
        }
    } else if constexpr (EPI == EPI_ADAM) {
        const int64_t moff = int64_t(b) * p.m_bstride + int64_t(row) * p.ldm + col0;
        const int64_t doff = int64_t(b) * p.d_bstride + int64_t(row) * p.ldd + col0;
        float* mm = p.mom_m + moff;
        float* vv = p.mom_v + moff;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            float4 m4 = *reinterpret_cast<const float4*>(mm + j);
            float4 v4 = *reinterpret_cast<const float4*>(vv + j);
            float* mp = &m4.x;
            float* vp = &v4.x;
            float4 h, l;
            float* hp = &h.x;
            float* lp = &l.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float g = p.alpha * __uint_as_float(r[j + e]);
                const float m = p.b1 * mp[e] + (1.f - p.b1) * g;
                const float v = p.b2 * vp[e] + (1.f - p.b2) * (g * g);
                mp[e] = m;
                vp[e] = v;
                const float s = (m * p.inv_bc1) / (sqrtf(v * p.inv_bc2) + p.adam_eps);
                out_split(p, s, hp[e], lp[e], p.Dlo != nullptr);
            }
            *reinterpret_cast<float4*>(mm + j) = m4;
            *reinterpret_cast<float4*>(vv + j) = v4;
            *reinterpret_cast<float4*>(p.Dhi + doff + j) = h;
            if (p.Dlo) *reinterpret_cast<float4*>(p.Dlo + doff + j) = l;
        }
    }
}

// EPI_APPLY, warp-cooperative: the warp's 32 rows x 32 columns go through a
// shared-memory transpose so that every read-modify-write of theta touches
// 32 consecutive floats of one row (one 128-byte line per instruction)
// instead of 32 rows (apply_update precond.cpp:244-251, NonFinite :248).
__device__ __forceinline__ void apply_chunk(const GemmParams& p, int b, int row0, int col0, const uint32_t (&r)[32],
                                            float (*scratch)[33]) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 32; ++j) scratch[lane][j] = p.alpha * __uint_as_float(r[j]);
    __syncwarp();
    const ApplyEntry e = p.apply[b];
    const int c = col0 + int(lane);
    bool bad = false;
    if (c < e.cols) {
        float* th = e.theta + c + int64_t(row0) * e.ld;
        const int rows = min(32, e.rows - row0);
        // all 32 loads in flight before any store (the warp covers 32 full 128-byte lines)
        float t[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) t[i] = (i < rows) ? __ldcs(th + int64_t(i) * e.ld) : 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            if (i < rows) {
                const float u = scratch[i][lane];
                const bool ok = isfinite(u);
                bad |= !ok;
                // a non-finite update element leaves theta unchanged (the reference
                // throws before touching theta, precond.cpp:248); the flag surfaces it
                __stcs(th + int64_t(i) * e.ld, ok ? t[i] - p.lr_eff * (u + p.wd * t[i]) : t[i]);
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0 && p.flag) atomicOr(p.flag, 1);
    __syncwarp();
}

// Coalesced STORE / SPLIT / SYM_EMA: the warp's 32 rows x 32 columns go
// through the shared-memory transpose, so every global access of a lane
// group is one 128-byte row segment (the row-per-thread mapping of
// epilogue_chunk touches 32 rows per instruction).
template <int EPI>
__device__ __forceinline__ void rows_chunk(const GemmParams& p, int b, int row0, int col0, const uint32_t (&r)[32],
                                           float (*scratch)[33]) {
    const uint32_t lane = threadIdx.x & 31;
    if constexpr (EPI == EPI_SYM_EMA) {
        if (row0 + 31 < col0) return;  // whole chunk strictly above the diagonal (warp-uniform)
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) scratch[lane][j] = p.alpha * __uint_as_float(r[j]);
    __syncwarp();
    const int c = col0 + int(lane);
    if constexpr (EPI == EPI_SPLIT || EPI == EPI_SPLIT2) {
        if (p.oscale) {  // fp16 (hi, lo) pairs at a scale fixed before the product (a bound on |D|)
            const float os = p.oscale[b];
            const int64_t o = int64_t(b) * p.d_bstride + int64_t(row0) * p.ldd + c;
            __half* dh = reinterpret_cast<__half*>(p.Dhi) + o;
            __half* dl = reinterpret_cast<__half*>(p.Dlo) + o;
#pragma unroll 8
            for (int i = 0; i < 32; ++i) {
                const float y = scratch[i][lane] * os;
                const __half h = __float2half_rn(y);
                dh[int64_t(i) * p.ldd] = h;
                dl[int64_t(i) * p.ldd] = __float2half_rn(y - __half2float(h));
            }
            if constexpr (EPI == EPI_SPLIT2) {
                const int64_t ot = int64_t(b) * p.d_bstride + int64_t(col0) * p.ldt + row0 + int(lane);
                __half* th = reinterpret_cast<__half*>(p.Thi) + ot;
                __half* tl = reinterpret_cast<__half*>(p.Tlo) + ot;
#pragma unroll 8
                for (int j = 0; j < 32; ++j) {
                    const float y = scratch[lane][j] * os;
                    const __half h = __float2half_rn(y);
                    th[int64_t(j) * p.ldt] = h;
                    tl[int64_t(j) * p.ldt] = __float2half_rn(y - __half2float(h));
                }
            }
            return;
        }
        if (p.omax) {  // per-batch max |D| for the next product's fp16 scale
            float mx = 0.f;
#pragma unroll 8
            for (int j = 0; j < 32; ++j) mx = fmaxf(mx, fabsf(scratch[lane][j]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (lane == 0) atomicMax(p.omax + b, __float_as_uint(mx));
        }
        float* dh = p.Dhi + int64_t(b) * p.d_bstride + int64_t(row0) * p.ldd + c;
        float* dl = p.Dlo ? p.Dlo + int64_t(b) * p.d_bstride + int64_t(row0) * p.ldd + c : nullptr;
#pragma unroll 8
        for (int i = 0; i < 32; ++i) {
            float h, l;
            out_split(p, scratch[i][lane], h, l, dl != nullptr);
            dh[int64_t(i) * p.ldd] = h;
            if (dl) dl[int64_t(i) * p.ldd] = l;
        }
        if constexpr (EPI == EPI_SPLIT2) {
            // D^T[col][row]: lanes = consecutive rows of one column (coalesced)
            float* th = p.Thi + int64_t(b) * p.d_bstride + int64_t(col0) * p.ldt + row0 + int(lane);
            float* tl = p.Tlo ? p.Tlo + int64_t(b) * p.d_bstride + int64_t(col0) * p.ldt + row0 + int(lane) : nullptr;
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {
                float h, l;
                out_split(p, scratch[lane][j], h, l, tl != nullptr);
                th[int64_t(j) * p.ldt] = h;
                if (tl) tl[int64_t(j) * p.ldt] = l;
            }
        }
    } else {
        float* cc = p.C + int64_t(b) * p.c_bstride + int64_t(row0) * p.ldc + c;
        if (p.beta != 0.f) {
            float o[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = cc[int64_t(i) * p.ldc];
#pragma unroll
            for (int i = 0; i < 32; ++i) scratch[i][lane] += p.beta * o[i];
        }
        if constexpr (EPI == EPI_STORE) {
#pragma unroll 8
            for (int i = 0; i < 32; ++i) cc[int64_t(i) * p.ldc] = scratch[i][lane];
        } else {  // SYM_EMA: lower triangle here, mirror below
#pragma unroll 8
            for (int i = 0; i < 32; ++i)
                if (row0 + i >= c) cc[int64_t(i) * p.ldc] = scratch[i][lane];
            __syncwarp();
            // mirror C[col][row] = C[row][col] for col < row; lanes = consecutive rows (coalesced)
            float* cb = p.C + int64_t(b) * p.c_bstride;
            const int row = row0 + int(lane);
#pragma unroll 8
            for (int j = 0; j < 32; ++j)
                if (row > col0 + j) cb[int64_t(col0 + j) * p.ldc + row] = scratch[lane][j];
        }
    }
    __syncwarp();
}

// EPI_ADAM, warp-cooperative (soap_scaled_step precond.cpp:213-221): the
// warp's 32 x 32 chunk of Ghat goes through the shared-memory transpose so
// that the moment read-modify-writes and the S stores are 128-byte coalesced
// rows; all 64 moment loads of a lane are in flight together.
__device__ __forceinline__ void adam_chunk(const GemmParams& p, int b, int row0, int col0, const uint32_t (&r)[32],
                                           float (*scratch)[33]) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 32; ++j) scratch[lane][j] = p.alpha * __uint_as_float(r[j]);
    __syncwarp();
    const int c = col0 + int(lane);
    float* mm = p.mom_m + int64_t(b) * p.m_bstride + int64_t(row0) * p.ldm + c;
    float* vv = p.mom_v + int64_t(b) * p.m_bstride + int64_t(row0) * p.ldm + c;
    float* dh = p.Dhi + int64_t(b) * p.d_bstride + int64_t(row0) * p.ldd + c;
    float* dl = p.Dlo ? p.Dlo + int64_t(b) * p.d_bstride + int64_t(row0) * p.ldd + c : nullptr;
#pragma unroll
    for (int h0 = 0; h0 < 32; h0 += 16) {  // two halves of 16 rows: 32 loads in flight per lane
        float mv[16], vvv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            mv[i] = __ldcs(mm + int64_t(h0 + i) * p.ldm);
            vvv[i] = __ldcs(vv + int64_t(h0 + i) * p.ldm);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float g = scratch[h0 + i][lane];
            const float m = p.b1 * mv[i] + (1.f - p.b1) * g;
            const float v = p.b2 * vvv[i] + (1.f - p.b2) * (g * g);
            __stcs(mm + int64_t(h0 + i) * p.ldm, m);
            __stcs(vv + int64_t(h0 + i) * p.ldm, v);
            float h, l;
            out_split(p, (m * p.inv_bc1) / (sqrtf(v * p.inv_bc2) + p.adam_eps), h, l, dl != nullptr);
            __stcs(dh + int64_t(h0 + i) * p.ldd, h);
            if (dl) __stcs(dl + int64_t(h0 + i) * p.ldd, l);
        }
    }
    __syncwarp();
}

// EPI_SYM_SPLIT / EPI_NS, warp-cooperative: the 32 x 32 chunk's lower
// triangle is written as (hi, lo) rows (coalesced) and mirrored to the upper
// triangle (lanes = consecutive rows: coalesced), so the output is exactly
// symmetric. EPI_NS also writes T = ns_a I - ns_b M the same way and folds
// max|M - I| into resid[b] (a non-finite M reports +inf).
template <bool NS>
__device__ __forceinline__ void sym_split_chunk(const GemmParams& p, int b, int row0, int col0,
                                                const uint32_t (&r)[32], float (*scratch)[33]) {
    const uint32_t lane = threadIdx.x & 31;
    if (row0 + 31 < col0) return;  // whole chunk strictly above the diagonal (warp-uniform)
#pragma unroll
    for (int j = 0; j < 32; ++j) scratch[lane][j] = p.alpha * __uint_as_float(r[j]);
    __syncwarp();
    const int64_t base = int64_t(b) * p.d_bstride;
    float* mh = p.Dhi + base;
    float* ml = p.Dlo ? p.Dlo + base : nullptr;
    float* th = NS ? p.Thi + base : nullptr;
    float* tl = (NS && p.Tlo) ? p.Tlo + base : nullptr;
    // fp16-pair outputs (oscale): M (and T) as scaled fp16 (hi, lo) __half arrays at the same offsets
    const float os = p.oscale ? p.oscale[b] : 0.f;
    __half* mh16 = reinterpret_cast<__half*>(p.Dhi) + base;
    __half* ml16 = reinterpret_cast<__half*>(p.Dlo) + base;
    __half* th16 = NS ? reinterpret_cast<__half*>(p.Thi) + base : nullptr;
    __half* tl16 = NS ? reinterpret_cast<__half*>(p.Tlo) + base : nullptr;
    float res = 0.f;
    auto put = [&](int64_t off, float v, bool diag) {
        if (p.oscale) {
            const float y = v * os;
            __half h = __float2half_rn(y);
            mh16[off] = h;
            ml16[off] = __float2half_rn(y - __half2float(h));
            if constexpr (NS) {
                const float t = ((diag ? p.ns_a : 0.f) - p.ns_b * v) * os;
                h = __float2half_rn(t);
                th16[off] = h;
                tl16[off] = __float2half_rn(t - __half2float(h));
            }
            return;
        }
        float h, l;
        out_split(p, v, h, l, ml != nullptr);
        mh[off] = h;
        if (ml) ml[off] = l;
        if constexpr (NS) {
            const float t = (diag ? p.ns_a : 0.f) - p.ns_b * v;
            out_split(p, t, h, l, tl != nullptr);
            th[off] = h;
            if (tl) tl[off] = l;
        }
    };
    const int c = col0 + int(lane);
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
        const int row = row0 + i;
        if (row >= c) {
            const float v = scratch[i][lane];
            put(int64_t(row) * p.ldd + c, v, row == c);
            if constexpr (NS) {
                const float d = fabsf(v - (row == c ? 1.f : 0.f));
                res = isfinite(v) ? fmaxf(res, d) : __int_as_float(0x7f800000);
            }
        }
    }
    __syncwarp();
    const int row = row0 + int(lane);
#pragma unroll 4
    for (int j = 0; j < 32; ++j)
        if (row > col0 + j) put(int64_t(col0 + j) * p.ldd + row, scratch[lane][j], false);
    if constexpr (NS) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) res = fmaxf(res, __shfl_xor_sync(0xffffffffu, res, o));
        if (lane == 0) atomicMax(p.resid + b, __float_as_uint(res));
    }
    __syncwarp();
}

template <int BN, int NPASS, int EPI, int CG = 1, bool SPL = false, bool F16 = false>
__global__ void __launch_bounds__(SPL ? 448 : 320, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                   const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl,
                   const __grid_constant__ GemmParams p) {
    using Cfg = GemmCfg<BN, NPASS, CG, SPL, F16>;
    static_assert(!F16 || (NPASS == 3 && !SPL), "3xFP16 takes (hi, lo) fp16 pairs from HBM");
    static_assert(!SPL || NPASS == 3, "the shared-memory split serves 3xTF32 only");
    constexpr int BM = Cfg::BM, BK = Cfg::BK, STAGES = Cfg::kStages;
    constexpr bool SPLIT = Cfg::kSplit;
    constexpr bool PAIR = CG == 2;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kRingBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* conv = tempty + 2;  // SPL: stage converted (the leader's: one arrive per CTA)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv + STAGES);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    float (*scratch)[33] = reinterpret_cast<float (*)[33]>(smem + Cfg::kRingBytes + 256 +
                                                           size_t(warp >= 2 ? warp - 2 : 0) * 32 * 33 * 4);
    // CTA pair: rank within the pair, the pair's index and count (tiles are
    // walked per pair; both CTAs decode the same tile sequence)
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    const int unit = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
    const int nunits = PAIR ? int(gridDim.x >> 1) : int(gridDim.x);

    // stage s: (A hi, A lo, B hi, B lo)
    auto a_hi = [&](int s) { return smem + size_t(s) * Cfg::kStageBytes; };
    auto a_lo = [&](int s) { return smem + size_t(s) * Cfg::kStageBytes + Cfg::kABytes; };
    auto b_hi = [&](int s) { return smem + size_t(s) * Cfg::kStageBytes + (SPLIT ? 2 : 1) * Cfg::kABytes; };
    auto b_lo = [&](int s) {
        return smem + size_t(s) * Cfg::kStageBytes + 2 * Cfg::kABytes + Cfg::kBBytes;
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmAh);
        tma_prefetch(&tmBh);
        if (SPLIT) {
            tma_prefetch(&tmAl);
            tma_prefetch(&tmBl);
        }
    }
    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);
            }
            for (int a = 0; a < 2; ++a) {
                mbar_init(&tfull[a], 1);
                // one arrive per epilogue warp (of both CTAs of a pair: the leader's barrier)
                mbar_init(&tempty[a], Cfg::kEpiWarps * CG);
            }
            if (SPL)
                for (int s = 0; s < STAGES; ++s) mbar_init(&conv[s], CG);
            fence_mbar_init();
        }
        __syncwarp();
        if constexpr (PAIR)
            tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
        else
            tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    }
    tc_fence_before();
    if constexpr (PAIR)
        cluster_sync();  // the peer's TMA and epilogue signal the leader's barriers: all initialised first
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int num_k = (p.K + BK - 1) / BK;  // F16: a K tail short of 64 is zero-filled by the TMA

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t full0 = PAIR ? mapa_shared(&full[0], 0) : 0u;
            for (int t = unit; t < p.num_tiles; t += nunits) {
                if (batch_skipped(p, t)) continue;
                int b, tm, tn;
                decode_tile(p, t, b, tm, tn);
                const int arow = tm * Cfg::TM + int(rank) * BM;
                const int brow = tn * BN + int(rank) * Cfg::kBRows;
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if constexpr (SPL) {
                        // local barrier: this CTA's converter warps split the raw operands
                        const uint32_t bytes = Cfg::kABytes * (p.a_raw ? 1 : 2) + Cfg::kBBytes * (p.b_raw ? 1 : 2);
                        mbar_arrive_expect_tx(&full[stage], bytes);
                        tma_load_3d(a_hi(stage), &tmAh, &full[stage], kb * BK, arow, b);
                        tma_load_3d(b_hi(stage), &tmBh, &full[stage], kb * BK, brow, b);
                        if (!p.a_raw) tma_load_3d(a_lo(stage), &tmAl, &full[stage], kb * BK, arow, b);
                        if (!p.b_raw) tma_load_3d(b_lo(stage), &tmBl, &full[stage], kb * BK, brow, b);
                    } else if constexpr (PAIR) {
                        // the leader's barrier expects both CTAs' bytes
                        if (rank == 0) mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes * 2);
                        const uint32_t fb = full0 + uint32_t(stage) * 8u;
                        tma_load_3d_pair(a_hi(stage), &tmAh, fb, kb * BK, arow, b);
                        tma_load_3d_pair(b_hi(stage), &tmBh, fb, kb * BK, brow, b);
                        if (SPLIT) {
                            tma_load_3d_pair(a_lo(stage), &tmAl, fb, kb * BK, arow, b);
                            tma_load_3d_pair(b_lo(stage), &tmBl, fb, kb * BK, brow, b);
                        }
                    } else {
                        mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
                        tma_load_3d(a_hi(stage), &tmAh, &full[stage], kb * BK, arow, b);
                        tma_load_3d(b_hi(stage), &tmBh, &full[stage], kb * BK, brow, b);
                        if (SPLIT) {
                            tma_load_3d(a_lo(stage), &tmAl, &full[stage], kb * BK, arow, b);
                            tma_load_3d(b_lo(stage), &tmBl, &full[stage], kb * BK, brow, b);
                        }
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = F16 ? idesc_f16(Cfg::TM, BN) : idesc_tf32(Cfg::TM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = unit; t < p.num_tiles; t += nunits) {
                if (batch_skipped(p, t)) continue;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + uint32_t(acc * BN);
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(SPL ? &conv[stage] : &full[stage], phase);
                    tc_fence_after();
                    const uint64_t ah = umma_desc_k_sw128(a_hi(stage));
                    const uint64_t bh = umma_desc_k_sw128(b_hi(stage));
                    const uint64_t al = SPLIT ? umma_desc_k_sw128(a_lo(stage)) : 0;
                    const uint64_t bl = SPLIT ? umma_desc_k_sw128(b_lo(stage)) : 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {  // four 32-byte K steps per 128-byte row
                        const uint64_t adv = uint64_t(k * 32) >> 4;  // 8 tf32 / 16 fp16 = 32 bytes along K
                        if constexpr (F16) {  // hi*hi + hi*lo + lo*hi, kind::f16
                            if constexpr (PAIR) {
                                mma_f16_pair(d, ah + adv, bh + adv, idesc, (kb | k) != 0 ? 1u : 0u);
                                mma_f16_pair(d, ah + adv, bl + adv, idesc, 1u);
                                mma_f16_pair(d, al + adv, bh + adv, idesc, 1u);
                            } else {
                                mma_f16(d, ah + adv, bh + adv, idesc, (kb | k) != 0 ? 1u : 0u);
                                mma_f16(d, ah + adv, bl + adv, idesc, 1u);
                                mma_f16(d, al + adv, bh + adv, idesc, 1u);
                            }
                            continue;
                        }
                        if constexpr (PAIR) {
                            mma_tf32_pair(d, ah + adv, bh + adv, idesc, (kb | k) != 0 ? 1u : 0u);
                            if (SPLIT) {
                                mma_tf32_pair(d, ah + adv, bl + adv, idesc, 1u);
                                mma_tf32_pair(d, al + adv, bh + adv, idesc, 1u);
                            }
                        } else {
                            mma_tf32(d, ah + adv, bh + adv, idesc, (kb | k) != 0 ? 1u : 0u);
                            if (SPLIT) {
                                mma_tf32(d, ah + adv, bl + adv, idesc, 1u);
                                mma_tf32(d, al + adv, bh + adv, idesc, 1u);
                            }
                        }
                    }
                    if constexpr (PAIR)
                        mma_commit_pair(&empty[stage], 0x3);  // both CTAs' stage is free
                    else
                        mma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if constexpr (PAIR)
                    mma_commit_pair(&tfull[acc], 0x3);  // both CTAs' accumulator halves are ready
                else
                    mma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (SPL && warp >= 2 + Cfg::kEpiWarps) {
        // converters: x -> (hi, lo) in place for the raw operands of each stage
        const int ct = threadIdx.x - 32 * (2 + Cfg::kEpiWarps);  // 0 .. 127
        const uint32_t conv0 = PAIR ? mapa_shared(&conv[0], 0) : 0u;
        int stage = 0;
        uint32_t phase = 0;
        for (int t = unit; t < p.num_tiles; t += nunits) {
            if (batch_skipped(p, t)) continue;
            for (int kb = 0; kb < num_k; ++kb) {
                mbar_wait(&full[stage], phase);
                // kind::tf32 reads the leading 19 bits of each operand word and drops
                // the low 13 (measured: tools/tf32_probe.py), so the raw fp32 word
                // already is the operand hi = trunc_tf32(x); only lo = rn_tf32(x - hi)
                // is written (|lo| < ulp_tf32(x): x = hi + lo to 2^-22 relative)
                auto split_region = [&](const uint8_t* hi, uint8_t* lo, uint32_t bytes) {
                    const uint32_t h0 = smem_u32(hi), l0 = smem_u32(lo);
                    // lo = rn_tf32(x - trunc_tf32(x)): integer round-half-away on the
                    // magnitude bits (cvt.rna.tf32.f32 without its special-value checks)
                    auto lo_of = [](uint32_t xb) {
                        const float r = __uint_as_float(xb) - __uint_as_float(xb & 0xffffe000u);
                        return (__float_as_uint(r) + 0x1000u) & 0xffffe000u;
                    };
                    // bytes / 16 is a multiple of 512: four 16-byte loads in flight per thread
                    for (uint32_t i0 = ct; i0 < bytes / 16; i0 += 512) {
                        uint32_t x[4][4];
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(x[u][0]), "=r"(x[u][1]), "=r"(x[u][2]), "=r"(x[u][3])
                                         : "r"(h0 + (i0 + 128u * u) * 16u));
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(l0 + (i0 + 128u * u) * 16u),
                                         "r"(lo_of(x[u][0])), "r"(lo_of(x[u][1])), "r"(lo_of(x[u][2])),
                                         "r"(lo_of(x[u][3]))
                                         : "memory");
                    }
                };
                if (p.a_raw) split_region(a_hi(stage), a_lo(stage), Cfg::kABytes);
                if (p.b_raw) split_region(b_hi(stage), b_lo(stage), Cfg::kBBytes);
                // generic-proxy smem writes -> visible to the tensor core's async proxy
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (ct == 0) {
                    if constexpr (PAIR)
                        mbar_arrive_remote(conv0 + uint32_t(stage) * 8u);
                    else
                        mbar_arrive(&conv[stage]);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else {
        const int q = warp & 3;           // TMEM lane quadrant this warp may access
        const int half = (warp - 2) >> 2;  // which of the quadrant's two warps: even / odd column chunks
        int acc = 0;
        uint32_t acc_phase = 0;
        const uint32_t tempty0 = PAIR ? mapa_shared(&tempty[0], 0) : 0u;
        for (int t = unit; t < p.num_tiles; t += nunits) {
            if (batch_skipped(p, t)) continue;
            int b, tm, tn;
            decode_tile(p, t, b, tm, tn);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int row0 = tm * Cfg::TM + int(rank) * BM + q * 32;
            const int row = row0 + int(lane);
            const float unscale = F16 ? 1.f / (p.ascale[b] * p.bscale[b]) : 1.f;  // exact (powers of two)
#pragma unroll 1
            for (int c = half; c < BN / 32; c += 2) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + c * 32), r);
                tmem_ld_wait();
                if constexpr (F16) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * unscale);
                }
                if constexpr (EPI == EPI_APPLY)
                    apply_chunk(p, b, row0, tn * BN + c * 32, r, scratch);
                else if constexpr (EPI == EPI_ADAM)
                    adam_chunk(p, b, row0, tn * BN + c * 32, r, scratch);
                else if constexpr (EPI == EPI_STORE || EPI == EPI_SPLIT || EPI == EPI_SPLIT2 || EPI == EPI_SYM_EMA)
                    rows_chunk<EPI>(p, b, row0, tn * BN + c * 32, r, scratch);
                else if constexpr (EPI == EPI_SYM_SPLIT || EPI == EPI_NS)
                    sym_split_chunk<EPI == EPI_NS>(p, b, row0, tn * BN + c * 32, r, scratch);
                else
                    epilogue_chunk<EPI>(p, b, row, tn * BN + c * 32, r);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR)
                    mbar_arrive_remote(tempty0 + uint32_t(acc) * 8u);
                else
                    mbar_arrive(&tempty[acc]);
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    if constexpr (PAIR) {
        // no CTA leaves while its peer may still signal its barriers or read its TMEM
        tc_fence_before();
        cluster_sync();
        if (warp == 1) {
            tc_fence_after();
            tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
        }
    } else {
        __syncthreads();
        if (warp == 1) {
            tc_fence_after();
            tmem_dealloc<Cfg::kTmemCols>(tmem_base);
        }
    }
}

}  // namespace asg
