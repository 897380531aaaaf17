// SPDX-License-Identifier: Apache-2.0
//
// Host-callable launchers for every device kernel of the optimizer step.
// Implemented in asg_kernels.cu; used by the runtime (asg_runtime.cpp).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "asg_gemm.cuh"

namespace asg {

// True the first time it is called for the current device with `bits`:
// function attributes (dynamic shared-memory limits) are per device.
inline bool first_on_device(std::atomic<uint64_t>& bits) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t b = uint64_t(1) << (dev & 63);
    return !(bits.fetch_or(b) & b);
}

// Process-wide count of kernels launched by this library.
uint64_t launch_count();
void count_launch(uint64_t n = 1);

// A slab operand for the TN GEMM: [batch][rows][K] fp32 pair (lo may be null
// in TF32 mode).
struct Operand {
    const float* hi;
    const float* lo;
    int rows;
    int K;
    // 3xFP16 operand: hi / lo point at [batch][rows][K] fp16 arrays (cast), scaled
    // by the per-batch power of two `scale` (GemmCfg F16, f16_scale)
    const float* scale = nullptr;
};

struct GemmLaunch {
    Operand A, B;
    int batch;
    int epi;                 // EpiKind
    GemmParams p;            // epilogue fields; shape/tile fields are filled by the launcher
    const int2* sym_tiles;   // non-null: symmetric (lower-triangle) schedule
    int sym_tiles_count;
};

// Picks the output tile width for an output with `n` columns (multiple of 128).
// tile width of an n x n symmetric output over `batch` matrices (its lower-triangle tile list)
int gemm_bn_for(int n, int batch);
// Builds the lower-triangle tile list for an n x n symmetric output with
// 128 x BN tiles. Returns the count; `out` may be null to query.
int gemm_sym_tile_list(int n, int bn, int2* out);
cudaError_t gemm_launch(const GemmLaunch& g, int precision, int num_sms, cudaStream_t stream);

// Block descriptors for the gather/scatter kernels.
struct BlockRef {
    const float* src;   // first element of the block in the caller's tensor
    float* dst;         // (scatter targets)
    int64_t ld;
    int32_t rows, cols;
};

// G (caller layout, scaled by *scale or scale_val) -> padded slabs
// Gh/Gl [b][M][N] and GTh/GTl [b][N][M] (tf32 hi/lo; lo null => TF32 mode).
// vec: every block row is 16-byte aligned (col offsets, ld, width % 4 == 0): 64x64 float4 tiles.
void launch_prep_grad(const BlockRef* blocks_dev, int nb, int M, int N, const float* scale_dev,
                      float scale_val, float* Gh, float* Gl, float* GTh, float* GTl,
                      cudaStream_t s, bool vec = false);
// Fills [nb][M][M] slabs with the padded identity (hi = I, lo = 0).
void launch_identity_split(float* hi, float* lo, int nb, int M, int m, cudaStream_t s);
// Fills [nb][M][M] fp32 with identity on the leading m x m (KL start) or zero.
void launch_identity_f32(float* a, int nb, int M, int m, float diag, cudaStream_t s);
// Sum of squares of a strided 2-D fp32 tensor into *acc (double), and
// non-finite flag.
void launch_sqnorm(const float* x, int64_t rows, int64_t cols, int64_t ld, double* acc, int* flag,
                   cudaStream_t s);
// Multi-tensor variant: one CTA per chunk [e0, e1) of a strided 2-D tensor.
struct SqChunk {
    const float* x;
    int64_t ld, cols, e0, e1;
};
void launch_sqnorm_multi(const SqChunk* chunks, int count, double* acc, int* flag, cudaStream_t s);
// clip scale from the accumulated squared norm (harness.cpp:219-223).
void launch_clip_scale(const double* sqnorm, double clip_norm, float* scale_out, cudaStream_t s);
// AdamW + apply for a 1-D/degenerate parameter (precond.cpp:229-251).
void launch_adamw_apply(float* theta, int64_t ld_t, const float* grad, int64_t ld_g, int64_t rows,
                        int64_t cols, float* m, float* v, const float* scale_dev, float scale_val,
                        float b1, float b2, float inv_bc1, float inv_bc2, float eps, float lr_eff,
                        float wd, int* flag, cudaStream_t s);

// One 1-D / degenerate parameter of the multi-tensor AdamW launch.
struct AdamEntry {
    float* theta;
    const float* grad;
    float* m;
    float* v;
    int64_t ld_t, ld_g, rows, cols;
};
void launch_adamw_multi(const AdamEntry* entries, int count, int64_t max_elems, float scale_val, float b1, float b2,
                        float inv_bc1, float inv_bc2, float eps, float lr_eff, float wd, int* flag, cudaStream_t s);

// Refresh path (fp64).
// Snapshot: [b][M][M] fp32 slab's leading m x m -> [b][m][m] fp64 (+ trace).
void launch_snapshot(const float* src, int nb, int M, int m, double* dst, cudaStream_t s);
// Batched symmetric eigendecomposition (values ascending, vectors as columns).
// `work` must hold nb*n*n doubles. `status` receives per-matrix codes.
void launch_sym_eig(const double* A, double* values, double* vectors, double* work, int nb, int n,
                    int* status, cudaStream_t s);
// eps[b] = damping * tr(A_b) / n  (relative_damping precond.cpp:121-125).
void launch_relative_damping(const double* A, int nb, int n, double damping, double* eps,
                             cudaStream_t s);
// W[b][i][j] = V[b][i][j] * (values[b][j] + eps[b])^power; sets status[b] to
// ASG_ERR_NOT_PSD if a damped eigenvalue is <= 0 (densela.hpp:274-278).
void launch_scale_columns(const double* V, const double* values, const double* eps, double power,
                          int nb, int n, double* W, int* status, cudaStream_t s);
// C[b] = alpha * op(A[b]) * op(B[b]) + beta*C[b], fp64 (CUDA cores).
void launch_dgemm(bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int64_t lda,
                  int64_t sa, const double* B, int64_t ldb, int64_t sb, double beta, double* C,
                  int64_t ldc, int64_t sc, int nb, cudaStream_t s);
// fp64 [b][n][n] (optionally symmetrized) -> padded fp32 hi/lo slabs [b][M][M]
// (and transposed copies if *_t non-null).
void launch_f64_to_split(const double* src, int nb, int n, int M, bool symmetrize, float* hi,
                         float* lo, float* hi_t, float* lo_t, cudaStream_t s);
// fp64 [b][rows][cols] <-> padded fp32 [b][R][C] slab.
void launch_f64_to_f32(const double* src, int nb, int rows, int cols, float* dst, int R, int Cc,
                       cudaStream_t s);
void launch_f32_to_f64(const float* src, int nb, int rows, int cols, int R, int Cc, double* dst,
                       cudaStream_t s);

void launch_square_f64(const double* a, double* out, int64_t n, cudaStream_t s);

// fp32-level refresh helpers (tensor-core transforms of the refresh).
// Elementwise hi/lo tf32 split of an fp32 array.
void launch_split_slab(const float* src, float* hi, float* lo, int64_t count, cudaStream_t s);
// dst = hi + lo (a pair stored as plain fp32, ASG_PREC_3XTF32_SMEM state).
void launch_merge_pair(const float* hi, const float* lo, float* dst, int64_t count, cudaStream_t s);
// [b][M][M] fp32 slab (leading m x m) -> [b][m][m] fp64, symmetrized (A + A^T)/2.
void launch_snapshot_sym(const float* src, int nb, int M, int m, double* dst, cudaStream_t s);
// dst[b] = split(op(src[b])^T) for [b][R][C] -> [b][C][R]; op = identity or
// elementwise square; src_lo may be null (plain fp32 source). R, C % 32 == 0.
void launch_transpose_split(const float* src_hi, const float* src_lo, int nb, int R, int C, float* dst_hi,
                            float* dst_lo, bool square, cudaStream_t s);
// Elementwise (hi + lo)^2, resplit.
void launch_square_split(const float* hi, const float* lo, float* out_hi, float* out_lo, int64_t count,
                         cudaStream_t s);
// W = V diag((lam + eps)^power) on split [b][D][D] slabs (columns >= n zeroed).
void launch_scale_columns_split(const float* Vh, const float* Vl, const double* values, const double* eps,
                                double power, int nb, int n, int D, float* Wh, float* Wl, int* status,
                                cudaStream_t s);
// eps[b] = damping * tr(A_b) / n from an fp32 slab [b][M][M].
void launch_relative_damping_f32(const float* A, int nb, int M, int n, double damping, double* eps, cudaStream_t s);

// X = (3 I - S) / 2 on the leading d x d of S = V^T V (Newton-Schulz polar step).
void launch_ns_x(const float* S, int nb, int d, int D, float* Xh, float* Xl, cudaStream_t s);

// Per-block status from a both-sides eigensolve: out[k] <- first failure of in[k], in[cnt+k].
void launch_merge_status(const int* in, int cnt, int* out, cudaStream_t s);

// 3xFP16 operands (GemmCfg F16): the power of two s with max|x| s in [2^14, 2^15)
// (1 for an all-zero or non-finite max), hi = rn_f16(x s), lo = rn_f16(x s - hi).
// Per-batch max |x| of [nb][per] fp32 slabs into amax (float bits; zeroed first).
void launch_absmax(const float* src, int nb, int64_t per, unsigned int* amax, cudaStream_t s);
// per-slot max column abs-sum (1-norm) of n x n fp32 slots, float bits
void launch_colabs_max(const float* src, int nb, int n, int64_t per, unsigned int* out, cudaStream_t s);
// out0[b] (= out1[b] when given) = fp16 scale of a product bounded by 2^15 n1[b] / ascale[b]
void launch_bound_scale(int nb, const float* ascale, const unsigned int* n1, float* out0, float* out1, cudaStream_t s);
// [nb][per] fp32 -> fp16 pairs hi16 / lo16 ([nb][per] each) and the scales.
void launch_to_f16pair(const float* src, const unsigned int* amax, int nb, int64_t per, void* hi16, void* lo16,
                       float* scale, cudaStream_t s);
// Gradient blocks (caller layout, times scale_val) -> fp16 pairs of G [b][M][N] and
// G^T [b][N][M] with per-block scales (a max pass over the blocks first).
// the same with the scale predicted from the previous step's max (pred, persistent per block;
// zero before the first step), this step's max fused into the pass (now), and the blocks whose
// prediction failed rewritten at the exact scale (fix: per-block flags); needs M, N % 64 == 0
// and 16-byte aligned gradient rows
void launch_prep_grad_f16_pred(const BlockRef* blocks_dev, int nb, int M, int N, float scale_val, unsigned int* pred,
                               unsigned int* now, int* fix, void* Gh16, void* Gl16, void* GTh16, void* GTl16,
                               float* gscale, cudaStream_t s);
void launch_prep_grad_f16(const BlockRef* blocks_dev, int nb, int M, int N, float scale_val, unsigned int* amax,
                          void* Gh16, void* Gl16, void* GTh16, void* GTl16, float* gscale, cudaStream_t s,
                          bool vec = false);

// Multi-GPU: pack owned block slices into a contiguous buffer and back.
void launch_pack_blocks(const BlockRef* blocks_dev, const int64_t* offsets_dev, int nb, float* out,
                        cudaStream_t s);
void launch_unpack_blocks(const BlockRef* blocks_dev, const int64_t* offsets_dev, int nb,
                          const float* in, cudaStream_t s);
// dst = scale * in (the reduced gradient segment -> the owned gradient slices)
void launch_unpack_scaled(const BlockRef* blocks_dev, const int64_t* offsets_dev, int nb, const float* in,
                          float scale, cudaStream_t s);

// Synthetic N(0, sigma^2) gradients into block views, Philox4x32-10 keyed (seed, step, key).
struct SynthBlock {
    float* dst;
    int64_t ld;
    int32_t rows, cols;
    float sigma;
    uint32_t key;
};
void launch_synth_normal(const SynthBlock* blocks_dev, int nb, int max_rows, int max_cols, uint64_t seed,
                         uint64_t step, cudaStream_t s);

}  // namespace asg
