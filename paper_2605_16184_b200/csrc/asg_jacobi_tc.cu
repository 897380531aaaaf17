// SPDX-License-Identifier: Apache-2.0
//
// Tensor-core block Jacobi: the batched symmetric eigensolver of the F32
// refresh (asg_refresh_mode F32), replacing sym_eig (densela.hpp:182-264) for
// factors above kSmallEighN. fp32-level arithmetic:
//
//   * A (the factor, rotated into the previous eigenbasis) and V (the
//     accumulated rotation) live in HBM as plain fp32, natural order; the
//     apply splits each operand chunk into (hi, lo) in shared memory.
//   * Columns are split into JW-wide blocks (32 below kWidePairN, 64 from
//     there); a round pairs the blocks by a round-robin tournament (m/2
//     disjoint pairs, m-1 rounds per sweep).
//   * tj_pair_kernel: one CTA per (matrix, pair) gathers the PW x PW pair
//     matrix (PW = 2 JW) and gives it one inner Jacobi sweep in shared memory
//     (fp32; odd-even ordering with one fused, conflict-free, load-batched
//     pass per round; for PW = 128 the pair rotation stays in registers;
//     ascending order within the pair = sorted block Jacobi); it writes J^T
//     as a split pair, or flags the pair as converged when no element exceeds
//     |a_ij| > tol * max(sqrt(a_ii a_jj), noise floor). Pairs with at most
//     kFewBig large elements rotate them one by one (classical Jacobi).
//   * tj_apply_kernel (tcgen05): every 128x128 tile (pair k1 rows, pair k2
//     columns, k1 <= k2: A stays exactly symmetric, so the epilogue writes the
//     transpose of an off-diagonal result into tile (k2, k1)) of A becomes
//     (J_k1^T A_tile) J_k2 -- two chained 3xTF32 MMAs: the first takes the
//     mirror tile A(k2, k1) as its K-major B operand, the intermediate Y stays
//     in TMEM (split in place into (Y_hi, Y_lo)) as the A operand of the
//     second -- and every 128-row panel of V becomes
//     V_tile J_k2. Tiles whose pairs are both converged are skipped (a CTA
//     with none left exits before allocating TMEM); tiles are pipelined
//     across the warp roles. All operand tiles are gathered by TMA (JW-row /
//     32-column boxes of the natural layout), so no data is permuted between
//     rounds.
//   * A sweep that rotated nothing ends the iteration (device flags; the
//     sweeps run in a CUDA-graph WHILE loop), within the reference's budget of
//     30 sweeps (densela.hpp:194); eigenvalues diag(A) are sorted ascending
//     with a stable index order (densela.hpp:251-262).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>
#include <mutex>
#include <tuple>

#include "../../include/asteria_b200.h"
#include "asg_eigh.cuh"
#include "asg_kernels.cuh"
#include "asg_ptx.cuh"

namespace asg {
namespace {

constexpr int JP = 128;  // apply tile: 128/PW pairs of two JW-wide blocks
// Pair width PW = 2 JW: 64 (tiles of two pairs) below kWidePairN, 128 (one
// pair per tile) from there on: small pairs make the shared-memory solves
// cheap, wide pairs halve the rounds (and the tensor-core work) per sweep.
// 512: measured faster than 1536 for warm refreshes (half the launches per
// sweep) and for cold solves at n = 512 and 1024 once the wide pair solve got
// faster (tools/gpu_wide.sh, gpu_wide2.sh).
constexpr int kWidePairN = 512;
constexpr int kFewBig = 8;  // pair solves with at most this many large elements rotate them one by one
// Pair-solve ordering: the odd-even ordering (one fused, conflict-free,
// load-batched pass per round) for both widths -- measured 2.3x (PW = 128) and
// 1.5x (PW = 64) faster than the round-robin ordering with separate row and
// column passes, which stays available (ASG_TJ_OE=0) for comparison.
constexpr int kOddEvenWide = 1, kOddEvenNarrow = 1;
// Rotation parameters in fp64 (ASG_TJ_ROT32=1: fp32, 6% faster pair solves at
// equal eigen-residuals, but the non-unit c^2+s^2 it leaves in the accumulated
// rotations moved the KL-Shampoo F32 trajectory test 1.7x past its tolerance).
constexpr int kRot32 = 0;
#ifndef ASG_TJ_SB
#define ASG_TJ_SB 4  // S items per load batch of the odd-even pass (2: same time, 8: 3-5% slower)
#endif
#ifndef ASG_TJ_NARROW_CTAS
#define ASG_TJ_NARROW_CTAS 4
#endif
constexpr int kNarrowPairCtas = ASG_TJ_NARROW_CTAS;  // resident narrow pair solves per SM (register cap)
constexpr int kInner = 1;  // inner sweeps of the pair solve (more outer sweeps are cheaper than inner ones)

__device__ __forceinline__ int tourney(int pos, int r, int P) { return pos == 0 ? 0 : 1 + (pos - 1 + r) % (P - 1); }
__device__ __forceinline__ void pair_of(int k, int r, int m, int& p, int& q) {
    p = tourney(k, r, m);
    q = tourney(m - 1 - k, r, m);
    if (p > q) {
        const int t = p;
        p = q;
        q = t;
    }
}
// Absolute floor of the rotation threshold, as a multiple of tol: the RMS
// eigenvalue ||A||_F / sqrt(n), raised to the fp32 rounding level of a factor
// accumulated over n-term sums (8 * 2^-24 * sqrt(n) of the RMS) so that pure
// rounding noise is never chased.
__device__ __forceinline__ float noise_floor(double fro, int n, float tol) {
    const double rms = fro / sqrt(double(n));
    const double lvl = 8.0 * 5.9604644775390625e-08 * sqrt(double(n));
    return float(rms * fmax(1.0, lvl / double(tol)));
}

// pair-local index -> natural index
template <int JW>
__device__ __forceinline__ int nat(int i, int p, int q) { return i < JW ? p * JW + i : q * JW + (i - JW); }

// ---- init -------------------------------------------------------------------
// ||B||_F^2, the Gershgorin bound (max absolute row sum) for the padding and
// a non-finite flag, accumulated with atomics; grid (D/32 row groups, nb),
// one warp per row, lanes along the row (coalesced).
__global__ void tj_stats_kernel(const float* __restrict__ B, int n, int D, double* __restrict__ fro2,
                                unsigned* __restrict__ bound_bits, int* __restrict__ bad) {
    const int64_t b = blockIdx.y;
    const float* Bb = B + b * int64_t(D) * D;
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    bool nf = false;
    for (int r = blockIdx.x * 32 + (threadIdx.x >> 5); r < min(n, blockIdx.x * 32 + 32); r += blockDim.x >> 5) {
        float rs = 0.f;
        for (int c = lane; c < n; c += 32) {
            const float x = Bb[int64_t(r) * D + c];
            nf |= !isfinite(x);
            s += double(x) * x;
            rs += fabsf(x);
        }
        for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffff, rs, o);
        if (lane == 0) atomicMax(&bound_bits[b], __float_as_uint(rs));  // non-negative: bit order = value order
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
    if (lane == 0 && s != 0.0) atomicAdd(&fro2[b], s);
    if (__any_sync(0xffffffff, nf) && lane == 0) atomicOr(&bad[b], 1);
}

__global__ void tj_stats_finish_kernel(int nb, double* __restrict__ fro, double* __restrict__ pad,
                                       const unsigned* __restrict__ bound_bits, const int* __restrict__ bad,
                                       int* __restrict__ active, int* __restrict__ status) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    fro[b] = sqrt(fro[b]);  // accumulated as ||B||_F^2
    const double mx = double(__uint_as_float(bound_bits[b]));
    pad[b] = mx > 0.0 ? 2.0 * mx : 1.0;
    active[b] = bad[b] ? 0 : 1;
    if (bad[b]) atomicCAS(&status[b], ASG_OK, ASG_ERR_NON_FINITE);
}

// A = (B + B^T)/2 (+ distinct padding diagonal above the spectrum), V = I;
// both split. Tiled 32x32 through shared memory so both reads are coalesced.
__global__ void tj_init_kernel(const float* __restrict__ B, int n, int D, const double* __restrict__ pad,
                               float* __restrict__ Ah, float* __restrict__ Al, float* __restrict__ Vh,
                               float* __restrict__ Vl) {
    __shared__ float t1[32][33], t2[32][33];
    const int64_t b = blockIdx.z;
    const int64_t DD = int64_t(D) * D;
    const int I = blockIdx.y * 32, J = blockIdx.x * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        t1[dy][threadIdx.x] = B[b * DD + int64_t(I + dy) * D + J + threadIdx.x];
        t2[dy][threadIdx.x] = B[b * DD + int64_t(J + dy) * D + I + threadIdx.x];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int i = I + dy, j = J + threadIdx.x;
        float x;
        if (i < n && j < n) x = 0.5f * (t1[dy][threadIdx.x] + t2[threadIdx.x][dy]);
        else x = (i == j) ? float(pad[b] * (1.0 + double(i - n + 1) * 1e-3)) : 0.f;
        // A and V are stored as plain fp32 in the Ah / Vh slabs (the apply splits
        // them in shared memory); the Al / Vl slabs are not used by the solve
        const int64_t o = b * DD + int64_t(i) * D + j;
        Ah[o] = x;
        Vh[o] = (i == j) ? 1.f : 0.f;
    }
}

// ---- pair solve -----------------------------------------------------------------
// One CTA per (pair k, matrix b): gathers the PW x PW pair matrix (blocks p,
// q), gives it one inner Jacobi sweep in shared memory and writes J^T into
// its diagonal PW x PW block of the 128x128 tile (for PW = 64 pairs 2g, 2g+1
// share a tile; the off-diagonal blocks stay zero).
template <int PW, int NT>
__global__ void __launch_bounds__(NT, PW == 64 ? kNarrowPairCtas : 1) tj_pair_kernel(const float* __restrict__ Ah, const float* __restrict__ Al,
                                                               int D, int m, int round, float* __restrict__ JTh,
                                                               float* __restrict__ JTl, int* __restrict__ pflag,
                                                               int* __restrict__ rotations,
                                                               const int* __restrict__ active,
                                                               const double* __restrict__ fro, int n, float tol,
                                                               int inner_sweeps, int oe_order, int rot32) {
    constexpr int JW = PW / 2, G = JP / PW;  // G pairs share one 128x128 tile
    extern __shared__ float tj_pair_smem[];
    float* S = tj_pair_smem;            // [PW][PW+1]
    float* Z = S + PW * (PW + 1);       // [PW][PW+1]
    __shared__ float cs[PW / 2], sn[PW / 2];
    __shared__ int pa[PW / 2], pc[PW / 2];
    __shared__ int rank_of[PW];
    const int k = blockIdx.x;
    const int64_t b = blockIdx.y;
    const int npairs = m / 2, ntiles = npairs / G;
    int* flag = pflag + b * npairs + k;
    if (!active[b]) {
        if (threadIdx.x == 0) *flag = 0;
        return;
    }
    int p, q;
    pair_of(k, round, m, p, q);
    const int64_t DD = int64_t(D) * D;
    for (int e = threadIdx.x; e < PW * PW; e += blockDim.x) {
        const int i = e / PW, j = e % PW;
        const int64_t off = b * DD + int64_t(nat<JW>(i, p, q)) * D + nat<JW>(j, p, q);
        S[i * (PW + 1) + j] = Ah[off];
        Z[i * (PW + 1) + j] = (i == j) ? 1.f : 0.f;
    }
    __syncthreads();
    const float floor_s = noise_floor(fro[b], n, tol);
    auto big = [&](int i, int j, float t) {
        return fabsf(S[i * (PW + 1) + j]) > t * fmaxf(sqrtf(fabsf(S[i * (PW + 1) + i] * S[j * (PW + 1) + j])), floor_s);
    };
    bool any = false;
    int nbig = 0;
    for (int e = threadIdx.x; e < PW * PW; e += blockDim.x) {
        const int i = e / PW, j = e % PW;
        if (j > i && big(i, j, tol)) {
            any = true;
            ++nbig;
        }
    }
    const int half = k % G;
    const int64_t tile = (b * ntiles + k / G) * int64_t(JP) * JP + int64_t(half * PW) * JP + half * PW;
    float* jh = JTh + tile;  // block origin inside the quad tile, row stride JP
    float* jl = JTl + tile;
    if (!__syncthreads_or(any)) {
        // converged pair: J = I (the apply still runs for quads whose other pair moves)
        for (int e = threadIdx.x; e < PW * PW; e += blockDim.x) {
            const int i = e / PW, j = e % PW;
            jh[int64_t(i) * JP + j] = (i == j) ? 1.f : 0.f;
            jl[int64_t(i) * JP + j] = 0.f;
        }
        if (threadIdx.x == 0) *flag = 0;
        return;
    }
    if (threadIdx.x == 0) *flag = 1;
    const float itol = 0.1f * tol;
    // Few large elements (a warm refresh): classical Jacobi on the largest one
    // at a time (a block-wide argmax, one rotation) instead of a full cyclic
    // sweep of PW-1 synchronised rounds.
    __shared__ int red_n[32];
    __shared__ float red_v[32];
    __shared__ int red_e[32];
    {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        int cnt = nbig;
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffff, cnt, o);
        if (lane == 0) red_n[wid] = cnt;
        __syncthreads();
        int total = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) total += red_n[w];
        __syncthreads();
        if (total <= kFewBig) {
            for (int it = 0; it < 4 * kFewBig; ++it) {
                float best = 0.f;
                int be = -1;
                for (int e = threadIdx.x; e < PW * PW; e += blockDim.x) {
                    const int i = e / PW, j = e % PW;
                    if (j <= i) continue;
                    const float thr = itol * fmaxf(sqrtf(fabsf(S[i * (PW + 1) + i] * S[j * (PW + 1) + j])), floor_s);
                    const float ratio = fabsf(S[i * (PW + 1) + j]) / thr;
                    if (ratio > 1.f && ratio > best) {
                        best = ratio;
                        be = e;
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const float ob = __shfl_xor_sync(0xffffffff, best, o);
                    const int oe = __shfl_xor_sync(0xffffffff, be, o);
                    if (ob > best) {
                        best = ob;
                        be = oe;
                    }
                }
                if (lane == 0) {
                    red_v[wid] = best;
                    red_e[wid] = be;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    float bb = 0.f;
                    int ee = -1;
                    for (int w = 0; w < int(blockDim.x >> 5); ++w)
                        if (red_v[w] > bb) {
                            bb = red_v[w];
                            ee = red_e[w];
                        }
                    red_e[0] = ee;
                    if (ee >= 0) {
                        const int a = ee / PW, c = ee % PW;
                        const double apq = S[a * (PW + 1) + c];
                        const double app = S[a * (PW + 1) + a], aqq = S[c * (PW + 1) + c];
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau)) : -1.0 / (-tau + sqrt(1.0 + tau * tau));
                        const double c1 = 1.0 / sqrt(1.0 + t * t);
                        cs[0] = float(c1);
                        sn[0] = float(t * c1);
                    }
                }
                __syncthreads();
                const int ee = red_e[0];
                if (ee < 0) break;
                const int a = ee / PW, c = ee % PW;
                const float cc = cs[0], ss = sn[0];
                for (int j = threadIdx.x; j < PW; j += blockDim.x) {  // rows a, c of S
                    const float x = S[a * (PW + 1) + j], y = S[c * (PW + 1) + j];
                    S[a * (PW + 1) + j] = cc * x - ss * y;
                    S[c * (PW + 1) + j] = ss * x + cc * y;
                }
                __syncthreads();
                for (int i = threadIdx.x; i < PW; i += blockDim.x) {  // columns a, c of S and Z
                    float x = S[i * (PW + 1) + a], y = S[i * (PW + 1) + c];
                    float na = cc * x - ss * y, nc = ss * x + cc * y;
                    if (i == a) nc = 0.f;
                    if (i == c) na = 0.f;
                    S[i * (PW + 1) + a] = na;
                    S[i * (PW + 1) + c] = nc;
                    x = Z[i * (PW + 1) + a];
                    y = Z[i * (PW + 1) + c];
                    Z[i * (PW + 1) + a] = cc * x - ss * y;
                    Z[i * (PW + 1) + c] = ss * x + cc * y;
                }
                __syncthreads();
            }
            inner_sweeps = 0;  // done: skip the cyclic sweep below
        }
    }
    // Odd-even ordering in position space: round r rotates the adjacent
    // position pairs (2k + r%2, 2k + 1 + r%2) and swaps every rotated pair's
    // two positions, so after PW rounds every two indices have met exactly
    // once (odd-even transposition of a reversed sequence). Pairs stay
    // adjacent, so one fused pass per round rotates each 2x2 block of S (rows
    // and columns) and the column pairs of Z with conflict-free shared-memory
    // access; the end state is a permutation of the eigenpairs, which the
    // ranking below absorbs. Odd rounds leave positions PW-1 and 0 idle; they
    // form the wrap "pair" k = PW/2-1 with the identity and no swap.
    if (oe_order && inner_sweeps > 0) {  // (a classical-path pair has already set inner_sweeps = 0)
        const int lane = threadIdx.x & 31;
        const bool flip = lane & 16;  // half-warps take the two rows in opposite order (banks)
        // Z lives in registers for the sweep: warp w owns rows [RPW w, RPW w + RPW),
        // lane l owns columns [CPL l, CPL l + CPL). Even rounds pair columns
        // inside a lane; odd rounds pair the lane's last column with the next
        // lane's first (one shuffle each way).
        // (wide pairs only: for PW = 64 the shuffle-per-odd-round layout measured
        // 11% slower than the shared-memory Z pass below)
        constexpr bool ZREG = PW == 128;
        constexpr int CPL = PW / 32, RPW = ZREG ? PW / (NT / 32) : 1;
        static_assert(CPL % 2 == 0 && (!ZREG || RPW * (NT / 32) == PW), "Z register layout");
        const int zrow0 = (threadIdx.x >> 5) * RPW, zcol0 = lane * CPL;
        float zr[RPW][CPL];
        if constexpr (ZREG) {
#pragma unroll
            for (int i = 0; i < RPW; ++i)
#pragma unroll
                for (int j = 0; j < CPL; ++j) zr[i][j] = (zrow0 + i == zcol0 + j) ? 1.f : 0.f;
        }
        for (int sweep = 0; sweep < inner_sweeps; ++sweep) {
            bool rot_any = false;
            for (int r = 0; r < PW; ++r) {
                const int odd = r & 1;
                if (threadIdx.x < PW / 2) {
                    const int kk = threadIdx.x;
                    const bool wrap = odd && kk == PW / 2 - 1;
                    const int a = 2 * kk + odd, c = wrap ? 0 : a + 1;
                    // Every pair's two positions swap after its rotation, so the
                    // idle wrap pair gets (c, s) = (0, 1): rotation + swap = diag(1, -1),
                    // an exact sign flip of position 0 -- the swaps stay unconditional.
                    float cc = wrap ? 0.f : 1.f, ss = wrap ? 1.f : 0.f;
                    if (!wrap && big(a, c, itol)) {
                        if (rot32) {  // fp32 rotation (the serial part of the round)
                            const float apq = S[a * (PW + 1) + c];
                            const float tau = (S[c * (PW + 1) + c] - S[a * (PW + 1) + a]) / (2.f * apq);
                            const float at = fabsf(tau);
                            const float t = at > 1e18f ? 0.5f / tau : copysignf(1.f, tau) / (at + sqrtf(fmaf(tau, tau, 1.f)));
                            cc = 1.f / sqrtf(fmaf(t, t, 1.f));
                            ss = t * cc;
                        } else {
                            // t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = u / v, written as
                            // sign(tau) |v| / (|u| + sqrt(u^2 + v^2)) (sign(tau) >= 0 for u == 0
                            // as before) in fp32: t only sets how well a_pq is annihilated (the
                            // pass zeroes it exactly); c = rsqrt(1 + t^2), s = t c in fp64 keep
                            // c^2 + s^2 = 1 to fp64 before the fp32 rounding. The round's
                            // serial chain: fp32 sqrt and division, one fp64 rsqrt (was three
                            // fp64 divisions and two fp64 square roots).
                            float v = 2.f * S[a * (PW + 1) + c];
                            float u = S[c * (PW + 1) + c] - S[a * (PW + 1) + a];
                            const float m = fmaxf(fabsf(u), fabsf(v));
                            if (m > 1e18f || m < 1e-18f) {  // t is scale-free: keep u^2 + v^2 finite
                                const int e = ilogbf(m);
                                u = ldexpf(u, -e);
                                v = ldexpf(v, -e);
                            }
                            const float r = sqrtf(fmaf(u, u, v * v));
                            const double t = double(copysignf(fabsf(v) / (fabsf(u) + r), (u == 0.f || (u > 0.f) == (v > 0.f)) ? 1.f : -1.f));
                            const double c1 = rsqrt(fma(t, t, 1.0));
                            cc = float(c1);
                            ss = float(t * c1);
                        }
                        rot_any = true;
                    }
                    cs[kk] = cc;
                    sn[kk] = ss;
                }
                __syncthreads();
                // S: 2x2 blocks (ki, kj); a warp covers one ki and 32 consecutive kj.
                // Every item of the thread is loaded before any is stored (the
                // compiler cannot reorder shared loads past shared stores), so
                // the round is one batch of independent loads, math, stores.
                constexpr int SI = (PW / 2) * (PW / 2) / NT;
                constexpr int SB = SI > ASG_TJ_SB ? ASG_TJ_SB : SI;  // S items per load batch
                static_assert(SI * NT == (PW / 2) * (PW / 2) && SI % SB == 0 && NT % (PW / 2) == 0, "thread count");
                // a thread's items share one column pair kj (item it: ki = ki0 + it NT/(PW/2)),
                // so the column rotation and offsets are per round, not per item
                const int ki0 = threadIdx.x / (PW / 2), kj = threadIdx.x % (PW / 2);
                const int aj = 2 * kj + odd;
                const int bo = (odd && kj == PW / 2 - 1) ? -(PW - 1) : 1;  // column bj relative to aj
                const float cj = cs[kj], sj = sn[kj];
                // item 0's row offsets (first = the row this lane loads first); item it
                // adds it * ISTEP; only the last item of the last ki0 holds the odd
                // rounds' wrap pair, whose second row is position 0, not PW
                constexpr int ISTEP = 2 * (NT / (PW / 2)) * (PW + 1);
                const int ra = 2 * ki0 + odd;
                const int base0 = (flip ? ra + 1 : ra) * (PW + 1) + aj, base1 = (flip ? ra : ra + 1) * (PW + 1) + aj;
                const bool wrap_item = odd && ki0 == NT / (PW / 2) - 1;  // (for it = SI - 1)
#pragma unroll
                for (int h = 0; h < SI / SB; ++h) {
                    float q[SB][4];
                    int o0[SB], o1[SB];  // offsets of (r0, aj) and (r1, aj)
#pragma unroll
                    for (int it = 0; it < SB; ++it) {
                        o0[it] = base0 + (h * SB + it) * ISTEP;
                        o1[it] = base1 + (h * SB + it) * ISTEP;
                        if (h * SB + it == SI - 1 && wrap_item) {
                            if (flip) o0[it] -= PW * (PW + 1);
                            else o1[it] -= PW * (PW + 1);
                        }
                        q[it][0] = S[o0[it]];
                        q[it][1] = S[o0[it] + bo];
                        q[it][2] = S[o1[it]];
                        q[it][3] = S[o1[it] + bo];
                    }
#pragma unroll
                    for (int it = 0; it < SB; ++it) {
                        const int ki = ki0 + (h * SB + it) * (NT / (PW / 2));
                        // slots: f = the row loaded first (ai, or bi on flip lanes), g = the
                        // other; negating s on flip lanes makes the row rotation
                        // order-agnostic: F = c f - s' g, G = s' f + c g. The
                        // unconditional swaps are slot exchanges: the first row's
                        // address takes G, columns aj <- X1 and bj <- X0.
                        const float f0 = q[it][0], f1 = q[it][1], g0 = q[it][2], g1 = q[it][3];
                        const float ci = cs[ki];
                        const float si = flip ? -sn[ki] : sn[ki];
                        const float F0 = ci * f0 - si * g0, F1 = ci * f1 - si * g1;
                        const float G0 = si * f0 + ci * g0, G1 = si * f1 + ci * g1;
                        const float r00 = sj * G0 + cj * G1, r01 = cj * G0 - sj * G1;  // first row's address
                        const float r10 = sj * F0 + cj * F1, r11 = cj * F0 - sj * F1;  // second row's
                        S[o0[it]] = r00;
                        S[o0[it] + bo] = r01;
                        S[o1[it]] = r10;
                        S[o1[it] + bo] = r11;
                    }
                }
                {
                    // the annihilated element of a rotated pair (not the wrap pair): the
                    // thread whose item is the diagonal block ki == kj zeroes its two
                    // off-diagonal slots after the item's own stores
                    constexpr int KS = NT / (PW / 2);
                    const int d = kj - ki0;
                    if (d >= 0 && d % KS == 0 && sn[kj] != 0.f && cs[kj] != 0.f) {
                        const int a0 = base0 + (d / KS) * ISTEP, a1 = base1 + (d / KS) * ISTEP;
                        S[flip ? a0 : a0 + 1] = 0.f;
                        S[flip ? a1 + 1 : a1] = 0.f;
                    }
                }
                // Z (registers): rotate + swap column pairs of the lane's rows
                if constexpr (!ZREG) {
                    // Z (shared): column pairs; a warp covers two rows x 16 pairs (row
                    // stride PW+1: banks differ); batches of loads before stores
                    constexpr int ZI = PW * (PW / 2) / NT, ZH = ZI > 8 ? ZI / 2 : ZI;
                    auto zoff = [&](int e, int& kk, int& dc) {
                        const int w = e >> 5, l = e & 31;
                        const int row = 2 * (w / (PW / 32)) + (l >> 4);
                        kk = (w % (PW / 32)) * 16 + (l & 15);
                        dc = (odd && kk == PW / 2 - 1) ? -(PW - 1) : 1;
                        return row * (PW + 1) + 2 * kk + odd;
                    };
#pragma unroll
                    for (int h = 0; h < ZI / ZH; ++h) {
                        float zq[ZH][2];
#pragma unroll
                        for (int it = 0; it < ZH; ++it) {
                            int kk, dc;
                            const int zo = zoff(threadIdx.x + (h * ZH + it) * NT, kk, dc);
                            zq[it][0] = Z[zo];
                            zq[it][1] = Z[zo + dc];
                        }
#pragma unroll
                        for (int it = 0; it < ZH; ++it) {
                            int kk, dc;
                            const int zo = zoff(threadIdx.x + (h * ZH + it) * NT, kk, dc);
                            const float x = zq[it][0], y = zq[it][1];
                            const float cc = cs[kk], ss = sn[kk];
                            Z[zo] = ss * x + cc * y;  // rotate, then swap the two positions
                            Z[zo + dc] = cc * x - ss * y;
                        }
                    }
                } else if (!odd) {
#pragma unroll
                    for (int j = 0; j < CPL; j += 2) {
                        const int kk = (zcol0 + j) >> 1;
                        const float cc = cs[kk], ss = sn[kk];
#pragma unroll
                        for (int i = 0; i < RPW; ++i) {
                            const float x = zr[i][j], y = zr[i][j + 1];
                            zr[i][j] = ss * x + cc * y;  // rotate, then swap the two positions
                            zr[i][j + 1] = cc * x - ss * y;
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 1; j + 1 < CPL; j += 2) {  // pairs inside the lane
                        const int kk = (zcol0 + j - 1) >> 1;
                        const float cc = cs[kk], ss = sn[kk];
#pragma unroll
                        for (int i = 0; i < RPW; ++i) {
                            const float x = zr[i][j], y = zr[i][j + 1];
                            zr[i][j] = ss * x + cc * y;  // rotate, then swap the two positions
                            zr[i][j + 1] = cc * x - ss * y;
                        }
                    }
                    // pair (zcol0 + CPL - 1, zcol0 + CPL) spans lanes l, l+1; lane 31's is the
                    // identity wrap pair (PW-1, 0), as is lane 0's incoming one
                    const int kl = (zcol0 + CPL - 2) >> 1;        // pair whose first column is mine
                    const int kr = (zcol0 - 2) >> 1;              // pair whose second column is mine
                    // (lane 0's incoming pair is the wrap pair: c = 0, s = 1 negates its column)
                    const float cl = cs[kl], sl = sn[kl];
                    const float crr = cs[lane > 0 ? kr : PW / 2 - 1], srr = sn[lane > 0 ? kr : PW / 2 - 1];
#pragma unroll
                    for (int i = 0; i < RPW; ++i) {
                        const float mine_last = zr[i][CPL - 1], mine_first = zr[i][0];
                        const float from_right = __shfl_down_sync(0xffffffffu, mine_first, 1);
                        const float from_left = __shfl_up_sync(0xffffffffu, mine_last, 1);
                        if (lane < 31) {  // I hold x (first column of pair kl); lane 31's is the wrap's x (kept)
                            const float x = mine_last, y = from_right;
                            zr[i][CPL - 1] = sl * x + cl * y;
                        }
                        {  // I hold y (second column of pair kr)
                            const float x = from_left, y = mine_first;
                            zr[i][0] = crr * x - srr * y;
                        }
                    }
                }
                __syncthreads();
            }
            if (!__syncthreads_or(rot_any)) break;
        }
        if constexpr (ZREG) {
#pragma unroll
            for (int i = 0; i < RPW; ++i)
#pragma unroll
                for (int j = 0; j < CPL; ++j) Z[(zrow0 + i) * (PW + 1) + zcol0 + j] = zr[i][j];
            __syncthreads();
        }
        inner_sweeps = 0;
    }
    for (int sweep = 0; sweep < inner_sweeps; ++sweep) {
        bool rot_any = false;
        for (int r = 0; r < PW - 1; ++r) {
            if (threadIdx.x < PW / 2) {
                int a, c;
                pair_of(threadIdx.x, r, PW, a, c);
                float cc = 1.f, ss = 0.f;
                if (big(a, c, itol)) {
                    const double apq = S[a * (PW + 1) + c];
                    const double app = S[a * (PW + 1) + a], aqq = S[c * (PW + 1) + c];
                    const double tau = (aqq - app) / (2.0 * apq);
                    const double t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau)) : -1.0 / (-tau + sqrt(1.0 + tau * tau));
                    const double c1 = 1.0 / sqrt(1.0 + t * t);
                    cc = float(c1);
                    ss = float(t * c1);
                    rot_any = true;
                }
                cs[threadIdx.x] = cc;
                sn[threadIdx.x] = ss;
                pa[threadIdx.x] = a;
                pc[threadIdx.x] = c;
            }
            // nearly diagonal pairs (warm refreshes) rotate in few rounds: skip the rest
            if (!__syncthreads_or(threadIdx.x < PW / 2 && sn[threadIdx.x] != 0.f)) continue;
            if constexpr (PW == 128) {
                // wide pairs: row pass then column pass (conflict-free rows; the
                // fused 2x2 pass scatters over banks at this width)
                for (int e = threadIdx.x; e < (PW / 2) * PW; e += blockDim.x) {  // rows of S
                    const int kk = e / PW, j = e % PW;
                    const float ss = sn[kk];
                    if (ss == 0.f) continue;
                    const int a = pa[kk], c = pc[kk];
                    const float cc = cs[kk];
                    const float x = S[a * (PW + 1) + j], y = S[c * (PW + 1) + j];
                    S[a * (PW + 1) + j] = cc * x - ss * y;
                    S[c * (PW + 1) + j] = ss * x + cc * y;
                }
                __syncthreads();
                for (int e = threadIdx.x; e < (PW / 2) * PW; e += blockDim.x) {  // columns of S
                    const int kk = e % (PW / 2), i = e / (PW / 2);
                    const float ss = sn[kk];
                    if (ss == 0.f) continue;
                    const int a = pa[kk], c = pc[kk];
                    const float cc = cs[kk];
                    const float x = S[i * (PW + 1) + a], y = S[i * (PW + 1) + c];
                    float na = cc * x - ss * y, nc = ss * x + cc * y;
                    if (i == a) nc = 0.f;
                    if (i == c) na = 0.f;
                    S[i * (PW + 1) + a] = na;
                    S[i * (PW + 1) + c] = nc;
                }
            } else {
                // One pass: every 2x2 block (rows of pair ki, columns of pair kj) of S
                // becomes R_ki^T S_block R_kj (half the shared-memory traffic of a row
                // pass followed by a column pass), and Z's columns rotate.
                for (int e = threadIdx.x; e < (PW / 2) * (PW / 2); e += blockDim.x) {
                    const int ki = e / (PW / 2), kj = e % (PW / 2);
                    const float si = sn[ki], sj = sn[kj];
                    if (si == 0.f && sj == 0.f) continue;
                    const float ci = cs[ki], cj = cs[kj];
                    const int ai = pa[ki], bi = pc[ki], aj = pa[kj], bj = pc[kj];
                    float s00 = S[ai * (PW + 1) + aj], s01 = S[ai * (PW + 1) + bj];
                    float s10 = S[bi * (PW + 1) + aj], s11 = S[bi * (PW + 1) + bj];
                    // rows: [r_a; r_b] <- [c r_a - s r_b; s r_a + c r_b]
                    float t00 = ci * s00 - si * s10, t01 = ci * s01 - si * s11;
                    float t10 = si * s00 + ci * s10, t11 = si * s01 + ci * s11;
                    // columns: [c_a, c_b] <- [c c_a - s c_b, s c_a + c c_b]
                    s00 = cj * t00 - sj * t01;
                    s01 = sj * t00 + cj * t01;
                    s10 = cj * t10 - sj * t11;
                    s11 = sj * t10 + cj * t11;
                    if (ki == kj && si != 0.f) s01 = s10 = 0.f;  // the annihilated pair
                    S[ai * (PW + 1) + aj] = s00;
                    S[ai * (PW + 1) + bj] = s01;
                    S[bi * (PW + 1) + aj] = s10;
                    S[bi * (PW + 1) + bj] = s11;
                }
            }
            for (int e = threadIdx.x; e < (PW / 2) * PW; e += blockDim.x) {  // columns of Z
                const int kk = e % (PW / 2), i = e / (PW / 2);
                const float ss = sn[kk];
                if (ss == 0.f) continue;
                const int a = pa[kk], c = pc[kk];
                const float cc = cs[kk];
                const float x = Z[i * (PW + 1) + a], y = Z[i * (PW + 1) + c];
                Z[i * (PW + 1) + a] = cc * x - ss * y;
                Z[i * (PW + 1) + c] = ss * x + cc * y;
            }
            __syncthreads();
        }
        if (!__syncthreads_or(rot_any)) break;
    }
    // ascending order within the pair (sorted block Jacobi)
    if (threadIdx.x < PW) {
        const int i = threadIdx.x;
        const float di = S[i * (PW + 1) + i];
        int r = 0;
        for (int j = 0; j < PW; ++j) {
            const float dj = S[j * (PW + 1) + j];
            r += (dj < di) || (dj == di && j < i);
        }
        rank_of[i] = r;
    }
    __syncthreads();
    // J[:, rank(c)] = Z[:, c]  ->  J^T[rank(c)][row] = Z[row][c]
    for (int e = threadIdx.x; e < PW * PW; e += blockDim.x) {
        const int c = e / PW, row = e % PW;
        float h, l;
        split_tf32(Z[row * (PW + 1) + c], h, l);
        jh[int64_t(rank_of[c]) * JP + row] = h;
        jl[int64_t(rank_of[c]) * JP + row] = l;
    }
}

// ---- apply (tcgen05) ------------------------------------------------------------------
struct TJApply {
    float *Ah, *Al, *Vh, *Vl;   // natural layout [nb][D][D]
    const int* pflag;           // [nb][m/2] per pair
    const int* active;          // [nb]
    int D, m, round, nb;
    int tilesA, tilesV;         // per matrix: T(T+1)/2 (upper triangle) and T^2, T = D/128
};

constexpr uint32_t kChunk = JP * 32 * 4;      // 128 rows x 32 fp32 = 16 KB
constexpr uint32_t kStage1 = 4 * kChunk;      // A hi/lo + J hi/lo
constexpr uint32_t kStage2 = 2 * kChunk;      // J_k1^T hi/lo
constexpr uint32_t kRegionS = 2 * kStage1;    // 128 KB: MMA1 ring, then X^T (4 chunks hi/lo)
constexpr uint32_t kRegionT = 2 * kStage2;    // 64 KB
constexpr int kMaxFlags = 4096;  // nb * pairs per launch (asserted by the launcher)
constexpr size_t kApplySmem = 1024 + size_t(kRegionS) + kRegionT + 128 + kMaxFlags * 4;

__device__ __forceinline__ void tj_decode(const TJApply& p, int t, int& b, bool& isA, int& i1, int& i2) {
    const int per = p.tilesA + p.tilesV;
    b = t / per;
    int l = t - b * per;
    const int np2 = p.D / JP;  // 128x128 tiles per matrix row
    if (l < p.tilesA) {
        // A is symmetric: only tiles i1 <= i2 are computed (row-major upper
        // triangle); the epilogue writes each off-diagonal result to both halves.
        isA = true;
        i1 = 0;
        while (l >= np2 - i1) {
            l -= np2 - i1;
            ++i1;
        }
        i2 = i1 + l;
    } else {
        isA = false;
        l -= p.tilesA;
        i1 = l / np2;  // 128-row panel of V
        i2 = l - i1 * np2;
    }
}

// lo = rn_tf32(x - trunc_tf32(x)) of a 16 KB operand chunk (elementwise, so the
// swizzle does not matter), by one warp: kind::tf32 reads each raw fp32 word
// as hi = trunc_tf32(x) (asg_gemm.cuh's in-smem split), so x = hi + lo to 2^-22.
__device__ __forceinline__ void tj_split_lo(const uint8_t* hi, uint8_t* lo, uint32_t lane) {
    const uint32_t h0 = smem_u32(hi), l0 = smem_u32(lo);
    auto lo_of = [](uint32_t xb) {
        const float r = __uint_as_float(xb) - __uint_as_float(xb & 0xffffe000u);
        return (__float_as_uint(r) + 0x1000u) & 0xffffe000u;
    };
    for (uint32_t i0 = lane; i0 < kChunk / 16; i0 += 128) {  // 4 16-byte loads in flight per lane
        uint32_t x[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(x[u][0]), "=r"(x[u][1]), "=r"(x[u][2]), "=r"(x[u][3])
                         : "r"(h0 + (i0 + 32u * u) * 16u));
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(l0 + (i0 + 32u * u) * 16u),
                         "r"(lo_of(x[u][0])), "r"(lo_of(x[u][1])), "r"(lo_of(x[u][2])), "r"(lo_of(x[u][3]))
                         : "memory");
    }
}

template <int JW>
__global__ void __launch_bounds__(192, 1)
    tj_apply_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                    const __grid_constant__ CUtensorMap tmVh, const __grid_constant__ CUtensorMap tmVl,
                    const __grid_constant__ CUtensorMap tmJh, const __grid_constant__ CUtensorMap tmJl,
                    const __grid_constant__ TJApply p) {
    extern __shared__ uint8_t tj_smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tj_smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* S = smem;
    uint8_t* T = smem + kRegionS;
    uint64_t* bars = reinterpret_cast<uint64_t*>(T + kRegionT);
    uint64_t* full1 = bars;        // [2]
    uint64_t* empty1 = bars + 2;   // [2]
    uint64_t* full2 = bars + 4;    // [2]
    uint64_t* empty2 = bars + 6;   // [2]
    // TMEM (512 columns): MMA1 outputs in two 128-column buffers used by
    // alternating tiles (MMA1 of tile u+1 runs while the epilogue drains tile u),
    // Y_lo at 256 and A' at 384 for A tiles. xdone / xfree are per buffer
    // (bars 8 / 14 and 11 / 15).
    uint64_t* xdone = bars + 8;    // MMA1 complete
    uint64_t* xready = bars + 9;   // Y split into (Y_hi, Y_lo) in TMEM (4 epilogue warps)
    uint64_t* adone = bars + 10;   // MMA2 complete
    uint64_t* xfree = bars + 11;   // buffer 0 done with (4 epilogue warps)
    uint64_t* afree = bars + 13;   // A' read out (4 epilogue warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    // per-pair flags and per-matrix activity, read once per launch (most tiles of
    // a warm refresh are skipped; a global load per tile would serialise them)
    constexpr int G = JP / (2 * JW), NB = JP / JW;  // pairs and blocks per tile
    int* sflag = reinterpret_cast<int*>(bars + 16);
    const int npairs = p.m / 2, ntiles = npairs / G;
    const int nflags = p.nb * npairs;
    for (int i = threadIdx.x; i < nflags; i += blockDim.x) sflag[i] = p.pflag[i] | (p.active[i / npairs] << 1);
    __syncthreads();
    const int total = p.nb * (p.tilesA + p.tilesV);
    {
        // A CTA without a moving tile this round (late sweeps of a warm refresh)
        // leaves before allocating TMEM or arming barriers.
        bool work = false;
        for (int t = blockIdx.x + int(threadIdx.x) * int(gridDim.x); t < total && !work;
             t += int(blockDim.x) * int(gridDim.x)) {
            int b, i1, i2;
            bool isA;
            tj_decode(p, t, b, isA, i1, i2);
            if (!(sflag[b * npairs] >> 1)) continue;
            for (int t2 = 0; t2 < G; ++t2)
                work |= (sflag[b * npairs + G * i2 + t2] & 1) || (isA && (sflag[b * npairs + G * i1 + t2] & 1));
        }
        if (!__syncthreads_or(work)) return;
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmAh);
        tma_prefetch(&tmAl);
        tma_prefetch(&tmVh);
        tma_prefetch(&tmVl);
        tma_prefetch(&tmJh);
        tma_prefetch(&tmJl);
    }
    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < 2; ++s) {
                mbar_init(&full1[s], 1);
                mbar_init(&empty1[s], 1);
                mbar_init(&full2[s], 1);
                mbar_init(&empty2[s], 1);
            }
            mbar_init(xdone, 1);
            mbar_init(bars + 14, 1);
            mbar_init(bars + 15, 4);
            mbar_init(xready, 4);
            mbar_init(adone, 1);
            mbar_init(xfree, 4);
            mbar_init(afree, 4);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t idesc = idesc_tf32(JP, JP);

    // Tiles are pipelined across the roles (no CTA-wide barrier per tile):
    //   * the producer runs ahead through the operand rings (shared memory only
    //     holds operands: the A-tile intermediate stays in TMEM);
    //   * MMA1(u+2) reuses tile u's buffer once the epilogue is done with it
    //     (xfree: after X(u) is stored, or after MMA2(u) read Y(u)); MMA2 writes
    //     A' once the previous A tile's A' has been read (afree).
    // Every role walks the same tile sequence, so each tracks the phase of
    // every barrier it waits on by counting.
    uint32_t ph_full1[2] = {0, 0}, ph_empty1[2] = {0, 0}, ph_full2[2] = {0, 0}, ph_empty2[2] = {0, 0};
    uint32_t ph_x = 0, ph_xr = 0, ph_a = 0, ph_xf = 0, ph_af = 0;  // ph_x / ph_xf: bit b = buffer b
    int nt = 0;  // tiles processed so far (the TMEM buffer of this tile is nt & 1)
    int use1[2] = {0, 0}, use2[2] = {0, 0};  // producer: number of fills of each stage so far
    bool a_seen = false;  // an A tile seen

    for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int b, i1, i2;
        bool isA;
        tj_decode(p, t, b, isA, i1, i2);
        // skip converged work (uniform across the CTA)
        if (!(sflag[b * npairs] >> 1)) continue;  // matrix converged
        int f2 = 0, f1 = 0;
#pragma unroll
        for (int t2 = 0; t2 < G; ++t2) {
            f2 |= sflag[b * npairs + G * i2 + t2] & 1;
            if (isA) f1 |= sflag[b * npairs + G * i1 + t2] & 1;
        }
        if (!f2 && !f1) continue;
        // the tile's JW-wide blocks: pair G*g + t -> blocks (2t, 2t+1)
        int blk1[NB], blk2[NB];
#pragma unroll
        for (int t2 = 0; t2 < G; ++t2) {
            pair_of(G * i2 + t2, p.round, p.m, blk2[2 * t2], blk2[2 * t2 + 1]);
            if (isA) pair_of(G * i1 + t2, p.round, p.m, blk1[2 * t2], blk1[2 * t2 + 1]);
            else blk1[2 * t2] = blk1[2 * t2 + 1] = 0;
        }
        const int jb2 = b * ntiles + i2, jb1 = b * ntiles + i1;
        const int tb = nt & 1;
        const uint32_t tbuf = tmem + uint32_t(tb * 128);  // MMA1 output (X or Y), double-buffered
        const uint32_t tylo = tmem + 256u, tap = tmem + 384u;  // Y_lo and A' (A tiles, single)
        uint64_t* xdone_b = tb ? bars + 14 : xdone;
        uint64_t* xfree_b = tb ? bars + 15 : xfree;

        if (warp == 0) {
            if (lane == 0) {
                // MMA1 operands, 4 K-chunks, ring of 2 stages. Slots: M-side hi, lo;
                // B-side hi, lo. A plain-fp32 operand leaves its lo slot to the MMA warp.
                //   V tile: V panel (M, fp32) x J_k2 (B, hi/lo)  -> X = V J_k2
                //   A tile: J_k1^T (M, hi/lo) x mirror tile A(k2, k1) (B = A_tile in
                //           K-major form, fp32)                   -> Y = J_k1^T A_tile
                for (int c = 0; c < 4; ++c) {
                    const int s = c & 1;
                    if (use1[s] > 0) {
                        mbar_wait(&empty1[s], ph_empty1[s]);
                        ph_empty1[s] ^= 1;
                    }
                    ++use1[s];
                    uint8_t* st = S + s * kStage1;
                    mbar_arrive_expect_tx(&full1[s], kStage1 - kChunk);
                    if (isA) {
                        tma_load_3d(st, &tmJh, &full1[s], c * 32, 0, jb1);
                        tma_load_3d(st + kChunk, &tmJl, &full1[s], c * 32, 0, jb1);
                        const int col = blk1[(c * 32) / JW] * JW + (c * 32) % JW;  // K-chunk c: 32 k1 columns
#pragma unroll
                        for (int rb = 0; rb < NB; ++rb)  // JW-row boxes: the k2 rows
                            tma_load_3d(st + 2 * kChunk + rb * (kChunk / NB), &tmAh, &full1[s], col, blk2[rb] * JW, b);
                    } else {
                        const int col = blk2[(c * 32) / JW] * JW + (c * 32) % JW;  // K-chunk c: 32 k2 columns
#pragma unroll
                        for (int rb = 0; rb < NB; ++rb)
                            tma_load_3d(st + rb * (kChunk / NB), &tmVh, &full1[s], col, i1 * JP + rb * JW, b);
                        tma_load_3d(st + 2 * kChunk, &tmJh, &full1[s], c * 32, 0, jb2);
                        tma_load_3d(st + 3 * kChunk, &tmJl, &full1[s], c * 32, 0, jb2);
                    }
                }
                if (isA) {  // MMA2 B operand: J_k2 chunks (hi, lo)
                    for (int c = 0; c < 4; ++c) {
                        const int s = c & 1;
                        if (use2[s] > 0) {
                            mbar_wait(&empty2[s], ph_empty2[s]);
                            ph_empty2[s] ^= 1;
                        }
                        ++use2[s];
                        uint8_t* st = T + s * kStage2;
                        mbar_arrive_expect_tx(&full2[s], kStage2);
                        tma_load_3d(st, &tmJh, &full2[s], c * 32, 0, jb2);
                        tma_load_3d(st + kChunk, &tmJl, &full2[s], c * 32, 0, jb2);
                    }
                }
            }
        } else if (warp == 1) {
            if (lane == 0 && nt >= 2) {  // the epilogue is done with the tile that last used this buffer
                mbar_wait(xfree_b, (ph_xf >> tb) & 1u);
                ph_xf ^= 1u << tb;
            }
            // MMA1 into the buffer (128 columns). The plain-fp32 operand's lo part is
            // written next to it by the warp while the previous chunk's MMAs run
            // (kind::tf32 reads the raw word as trunc_tf32(x)).
            for (int c = 0; c < 4; ++c) {
                const int s = c & 1;
                mbar_wait(&full1[s], ph_full1[s]);
                ph_full1[s] ^= 1;
                uint8_t* st = S + s * kStage1;
                if (isA) tj_split_lo(st + 2 * kChunk, st + 3 * kChunk, lane);
                else tj_split_lo(st, st + kChunk, lane);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    tc_fence_after();
                    const uint64_t ah = umma_desc_k_sw128(st), al = umma_desc_k_sw128(st + kChunk);
                    const uint64_t bh = umma_desc_k_sw128(st + 2 * kChunk), bl = umma_desc_k_sw128(st + 3 * kChunk);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t adv = uint64_t(kk * 32) >> 4;
                        mma_tf32(tbuf, ah + adv, bh + adv, idesc, (c | kk) != 0 ? 1u : 0u);
                        mma_tf32(tbuf, ah + adv, bl + adv, idesc, 1u);
                        mma_tf32(tbuf, al + adv, bh + adv, idesc, 1u);
                    }
                    mma_commit(&empty1[s]);
                }
                __syncwarp();
            }
            if (lane == 0) {
                mma_commit(xdone_b);
                if (isA) {
                    // MMA2: A' = Y J_k2 with A = (Y_hi, Y_lo) read from TMEM (the epilogue
                    // split Y in place), B = J_k2 chunks from ring T
                    mbar_wait(xready, ph_xr);
                    ph_xr ^= 1;
                    if (a_seen) {  // A' of the previous A tile has been read out
                        mbar_wait(afree, ph_af);
                        ph_af ^= 1;
                    }
                    a_seen = true;
                    tc_fence_after();
                    for (int c = 0; c < 4; ++c) {
                        const int s = c & 1;
                        mbar_wait(&full2[s], ph_full2[s]);
                        ph_full2[s] ^= 1;
                        tc_fence_after();
                        uint8_t* st = T + s * kStage2;
                        const uint64_t bh = umma_desc_k_sw128(st), bl = umma_desc_k_sw128(st + kChunk);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t adv = uint64_t(kk * 32) >> 4;
                            const uint32_t k0 = uint32_t(c * 32 + kk * 8);
                            mma_tf32_ts(tap, tbuf + k0, bh + adv, idesc, (c | kk) != 0 ? 1u : 0u);
                            mma_tf32_ts(tap, tbuf + k0, bl + adv, idesc, 1u);
                            mma_tf32_ts(tap, tylo + k0, bh + adv, idesc, 1u);
                        }
                        mma_commit(&empty2[s]);
                    }
                    mma_commit(adone);
                }
            }
        } else {
            const int qd = warp & 3;  // TMEM lane quadrant: rows 32*qd .. 32*qd+31
            const int row = qd * 32 + int(lane);
            const uint32_t lq = uint32_t(qd * 32) << 16;
            mbar_wait(xdone_b, (ph_x >> tb) & 1u);
            ph_x ^= 1u << tb;
            tc_fence_after();
            if (isA) {
                // Y -> (Y_hi in place, Y_lo), the A operand pair of MMA2
#pragma unroll 1
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t r[32], lo[32];
                    tmem_ld_32x32b_x32(tbuf + lq + uint32_t(cc * 32), r);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        float h, l;
                        split_tf32(__uint_as_float(r[j]), h, l);
                        r[j] = __float_as_uint(h);
                        lo[j] = __float_as_uint(l);
                    }
                    tmem_st_32x32b_x32(tbuf + lq + uint32_t(cc * 32), r);
                    tmem_st_32x32b_x32(tylo + lq + uint32_t(cc * 32), lo);
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(xready);
                mbar_wait(adone, ph_a);
                ph_a ^= 1;
                tc_fence_after();
                // A' rows -> natural positions
                const int gr = blk1[row / JW] * JW + row % JW;
                const int64_t base = int64_t(b) * p.D * p.D + int64_t(gr) * p.D;
#pragma unroll 1
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tap + lq + uint32_t(cc * 32), r);
                    tmem_ld_wait();
                    const int gc = blk2[(cc * 32) / JW] * JW + (cc * 32) % JW;
                    float* dh = p.Ah + base + gc;  // A is plain fp32 (the Al slab is not used by the solve)
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<float4*>(dh + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                                         __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                    if (i1 != i2) {
                        // mirror tile (i2, i1): column gc + j of these rows becomes row gc + j;
                        // a warp's 32 rows are consecutive (one JW block), so each store is 128 B
                        const int64_t tb2 = int64_t(b) * p.D * p.D + int64_t(gc) * p.D + gr;
#pragma unroll
                        for (int j = 0; j < 32; ++j) p.Ah[tb2 + int64_t(j) * p.D] = __uint_as_float(r[j]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(afree);
                    mbar_arrive(xfree_b);  // MMA2 (complete: adone) was the last reader of Y
                }
            } else {
                const int gr = i1 * JP + row;
                const int64_t base = int64_t(b) * p.D * p.D + int64_t(gr) * p.D;
#pragma unroll 1
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tbuf + lq + uint32_t(cc * 32), r);
                    tmem_ld_wait();
                    const int gc = blk2[(cc * 32) / JW] * JW + (cc * 32) % JW;
                    float* dh = p.Vh + base + gc;  // V is plain fp32 (the Vl slab is not used by the solve)
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<float4*>(dh + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                                         __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(xfree_b);
            }
        }
        ++nt;
    }
    // the epilogue warps waited for every MMA of their last tile: TMEM is idle
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

__global__ void tj_fill_status_kernel(int* status, int nb, int code) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nb) status[b] = code;
}

// ---- convergence / loop / finish ------------------------------------------------------
// Convergence test over the whole matrix (the pair kernels' skip rule applied
// to every off-diagonal element): big[b] = 1 if some element of matrix b still
// exceeds the threshold. Grid (D/32 row groups, nb).
__global__ void tj_check_kernel(const float* __restrict__ Ah, const float* __restrict__ Al, int D, int n,
                                const double* __restrict__ fro, const int* __restrict__ active, int* __restrict__ big,
                                float tol) {
    extern __shared__ float dgs[];  // |diag(A)| of matrix b
    const int64_t b = blockIdx.y;
    if (!active[b]) return;
    const int64_t DD = int64_t(D) * D;
    for (int i = threadIdx.x; i < D; i += blockDim.x)
        dgs[i] = fabsf(Ah[b * DD + int64_t(i) * D + i]);
    __syncthreads();
    const float floor_s = noise_floor(fro[b], n, tol);
    bool any = false;
    for (int r = blockIdx.x * 32 + (threadIdx.x >> 5); r < min(D, blockIdx.x * 32 + 32); r += blockDim.x >> 5) {
        const float dr = dgs[r];
        // upper triangle only: the pair kernels test a_ij with i < j too (the two
        // triangles differ in their last bits after independent tile products)
        for (int c = r + 1 + (threadIdx.x & 31); c < D; c += 32) {
            const int64_t o = b * DD + int64_t(r) * D + c;
            const float x = fabsf(Ah[o]);
            if (x == 0.f) continue;
            const float dc = dgs[c];
            any |= x > tol * fmaxf(sqrtf(dr * dc), floor_s);
        }
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) big[b] = 1;
}

// After a sweep: a matrix stays active only while the check found a large element.
__global__ void tj_settle_kernel(int nb, int* __restrict__ active, int* __restrict__ big, int* __restrict__ sweeps,
                                 int debug, int n, int count_sweep) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb || !active[b]) return;
    if (count_sweep) sweeps[b] += 1;
    if (debug) printf("tjdbg n=%d b=%d sweeps=%d still_large=%d\n", n, b, sweeps[b], big[b]);
    if (!big[b]) active[b] = 0;
    big[b] = 0;
}

__global__ void tj_loop_kernel(const int* __restrict__ active, int nb, int* __restrict__ sweep_count, int max_sweeps,
                               cudaGraphConditionalHandle handle) {
    int any = 0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) any |= active[b];
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) {
        const int s = ++*sweep_count;
        cudaGraphSetConditional(handle, (any && s < max_sweeps) ? 1u : 0u);
    }
}

// One CTA per matrix: ascending ranks of diag(A) (stable by index); the n real
// eigenvalues come first (padding sits above the spectrum).
__global__ void tj_rank_kernel(const float* __restrict__ Ah, const float* __restrict__ Al, int n, int D,
                               int* __restrict__ rank, double* __restrict__ values, const int* __restrict__ active,
                               int* __restrict__ status, const int* __restrict__ sweeps, int* __restrict__ ident) {
    extern __shared__ float dg[];
    const int64_t b = blockIdx.x;
    const int64_t DD = int64_t(D) * D;
    for (int i = threadIdx.x; i < D; i += blockDim.x) dg[i] = Ah[b * DD + int64_t(i) * D + i];
    __syncthreads();
    if (threadIdx.x == 0 && active[b]) atomicCAS(&status[b], ASG_OK, ASG_ERR_NO_CONVERGENCE);
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
        const float di = dg[i];
        int r = 0;
        for (int j = 0; j < D; ++j) {
            const float dj = dg[j];
            r += (dj < di) || (dj == di && j < i);
        }
        rank[b * D + r] = i;  // inverse permutation: output column r <- V column i
        if (r < n) values[b * n + r] = double(di);
    }
    // J = I exactly: no sweep rotated anything and the order is already ascending
    if (ident) {
        bool moved = false;
        for (int i = threadIdx.x; i < D; i += blockDim.x) {
            const float di = dg[i];
            for (int j = i + 1; j < D && !moved; ++j) moved |= dg[j] < di;  // a later smaller value reorders
        }
        const int any_moved = __syncthreads_or(moved);
        if (threadIdx.x == 0) ident[b] = (!any_moved && sweeps[b] == 0) ? 1 : 0;
    }
}

// J[i][r] = V[i][src(r)] for i, r < n (zero elsewhere), split; src = the
// inverse rank permutation (coalesced writes; J^T follows by a tiled transpose).
__global__ void tj_gather_kernel(const float* __restrict__ Vh, const float* __restrict__ Vl,
                                 const int* __restrict__ src, int n, int D, float* __restrict__ Jh,
                                 float* __restrict__ Jl) {
    const int64_t b = blockIdx.y;
    const int64_t DD = int64_t(D) * D;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < DD; e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e / D), r = int(e % D);
        float h = 0.f, l = 0.f;
        if (i < n && r < n) {
            const int64_t o = b * DD + int64_t(i) * D + src[b * D + r];
            split_tf32(Vh[o], h, l);  // V is plain fp32
        }
        Jh[b * DD + e] = h;
        if (Jl) Jl[b * DD + e] = l;
    }
}

// Rayleigh-quotient eigenvalues and unit eigenvectors from the solve's J and
// W = B J (one 3xTF32 product): lambda_i = (J_i . W_i) / (J_i . J_i), then
// J_i /= |J_i|. This removes the slow drift of |J_i| and diag(A) that the
// tensor cores' fp32 accumulation leaves over hundreds of rotation products.
// Grid (D/32 column groups, nb), 256 threads = 32 columns x 8 row phases.
// Matrices that took no sweep (sweeps[b] == 0) have J = a permutation (the
// sort) and skipped the W = B J GEMM: their quotient is B's diagonal, read
// through J (j_i = e_src(i): sum_k J[k][i]^2 B[k][k] = B[src][src]).
__global__ void tj_rayleigh_kernel(float* __restrict__ Jh, float* __restrict__ Jl, float* __restrict__ JTh,
                                   float* __restrict__ JTl, const float* __restrict__ W, int n, int D,
                                   double* __restrict__ values, const float* __restrict__ B, int ldb,
                                   const int* __restrict__ sweeps) {
    __shared__ double sjw[8][32], sjj[8][32];
    __shared__ float scale[32];
    const int64_t b = blockIdx.y;
    const int64_t DD = int64_t(D) * D;
    const int cl = threadIdx.x & 31, ph = threadIdx.x >> 5;
    const int c = blockIdx.x * 32 + cl;
    double jw = 0.0, jj = 0.0;
    const bool perm = sweeps[b] == 0;
    for (int k = ph; k < n; k += 8) {
        const int64_t o = b * DD + int64_t(k) * D + c;
        const double j = double(Jh[o]) + (Jl ? double(Jl[o]) : 0.0);
        jw += perm ? (j == 0.0 ? 0.0 : j * j * double(B[b * int64_t(ldb) * ldb + int64_t(k) * ldb + k]))
                   : j * double(W[o]);
        jj += j * j;
    }
    sjw[ph][cl] = jw;
    sjj[ph][cl] = jj;
    __syncthreads();
    if (ph == 0) {
        double a = 0.0, q = 0.0;
        for (int t = 0; t < 8; ++t) {
            a += sjw[t][cl];
            q += sjj[t][cl];
        }
        float sc = 1.f;
        if (c < n && q > 0.0) {
            values[b * n + c] = a / q;
            sc = float(1.0 / sqrt(q));
        }
        scale[cl] = sc;
    }
    __syncthreads();
    // J[:, c] *= scale  (rows k, 32 consecutive columns per row)
    for (int k = ph; k < n; k += 8) {
        const int64_t o = b * DD + int64_t(k) * D + c;
        float h, l;
        split_tf32((Jh[o] + (Jl ? Jl[o] : 0.f)) * scale[cl], h, l);
        Jh[o] = h;
        if (Jl) Jl[o] = l;
    }
    // J^T rows [32 blockIdx.x, +32): row r scaled by scale[r - 32 blockIdx.x]
    for (int rr = ph; rr < 32; rr += 8) {
        const int r = blockIdx.x * 32 + rr;
        if (r >= n) continue;
        for (int k = cl; k < n; k += 32) {
            const int64_t o = b * DD + int64_t(r) * D + k;
            float h, l;
            split_tf32((JTh[o] + (JTl ? JTl[o] : 0.f)) * scale[rr], h, l);
            JTh[o] = h;
            if (JTl) JTl[o] = l;
        }
    }
}

// Ascending order of the refined values (ties/inversions at rounding level;
// the vectors keep their diag(A) order, which agrees to that level).
__global__ void tj_sort_values_kernel(double* __restrict__ values, int n) {
    extern __shared__ double sv[];
    const int64_t b = blockIdx.x;
    for (int i = threadIdx.x; i < n; i += blockDim.x) sv[i] = values[b * n + i];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double vi = sv[i];
        int r = 0;
        for (int j = 0; j < n; ++j) r += (sv[j] < vi) || (sv[j] == vi && j < i);
        values[b * n + r] = vi;
    }
}

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled tj_encode_fn() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(ptr);
    });
    return fn;
}

// 3-D map over [batch][rows][cols] fp32, box (32 cols x box_rows x 1), 128B swizzle.
bool tj_map(CUtensorMap* map, const float* base, int cols, int rows, int batch, int box_rows) {
    PFN_encodeTiled enc = tj_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {cuuint64_t(cols), cuuint64_t(rows), cuuint64_t(batch)};
    cuuint64_t strides[2] = {cuuint64_t(cols) * 4, cuuint64_t(cols) * cuuint64_t(rows) * 4};
    cuuint32_t box[3] = {32, cuuint32_t(box_rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

size_t tc_eigh_workspace_floats(int nb, int n) {
    const int D = (n + JP - 1) / JP * JP;
    const int m = D / 32;  // the narrow variant has the most pairs
    // A hi/lo, V hi/lo, J^T hi/lo per 128x128 tile, then per matrix: fro, pad (2 doubles = 4 floats),
    // active, sweeps, rotations, flags (m/2 pairs), ranks (D); and the loop counter.
    return size_t(nb) * (4 * size_t(D) * D + 2 * size_t(D / JP) * JP * JP + 4 + 3 + size_t(m / 2) + D) + 4;
}

int tc_eigh_dim(int n) { return (n + JP - 1) / JP * JP; }

namespace {
void tc_eigh_chunk(const float* B, int D_in, double* values, float* Jh, float* Jl, float* JTh, float* JTl, float* ws,
                   int nb, int n, int* status, int num_sms, cudaStream_t s, double tol, bool orthonormalize, int* ident) {
    const int D = (n + JP - 1) / JP * JP;
    (void)D_in;  // B, J, J^T are [nb][D][D] with D = roundup(n, 128) (== the group's padded dim)
    static const int wide_n = getenv("ASG_TJ_WIDE_N") ? atoi(getenv("ASG_TJ_WIDE_N")) : kWidePairN;  // tuning
    const bool wide = n >= wide_n;
    const int JW = wide ? 64 : 32;
    const int m = D / JW, npairs = m / 2, ntiles = D / JP;  // 128x128 J tiles per matrix
    const size_t DD = size_t(D) * D;
    float* Ah = ws;
    float* Al = Ah + size_t(nb) * DD;
    float* Vh = Al + size_t(nb) * DD;
    float* Vl = Vh + size_t(nb) * DD;
    float* JPh = Vl + size_t(nb) * DD;
    float* JPl = JPh + size_t(nb) * ntiles * JP * JP;
    double* fro = reinterpret_cast<double*>(JPl + size_t(nb) * ntiles * JP * JP);
    double* pad = fro + nb;
    int* active = reinterpret_cast<int*>(pad + nb);
    int* sweeps = active + nb;
    int* rotations = sweeps + nb;
    int* pflag = rotations + nb;
    int* rank = pflag + size_t(nb) * npairs;
    int* loop_count = rank + size_t(nb) * D;

    static std::atomic<uint64_t> attr_bits{0};
    if (first_on_device(attr_bits)) {
        cudaFuncSetAttribute(tj_apply_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kApplySmem));
        cudaFuncSetAttribute(tj_apply_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kApplySmem));
        cudaFuncSetAttribute(tj_pair_kernel<64, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 65 * 4);
        cudaFuncSetAttribute(tj_pair_kernel<128, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 128 * 129 * 4);
        cudaFuncSetAttribute(tj_pair_kernel<128, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 128 * 129 * 4);
        cudaFuncSetAttribute(tj_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 4);
        cudaFuncSetAttribute(tj_sort_values_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 8);
    }
    TJApply ap{};
    ap.Ah = Ah;
    ap.Al = Al;
    ap.Vh = Vh;
    ap.Vl = Vl;
    ap.pflag = pflag;
    ap.active = active;
    ap.D = D;
    ap.m = m;
    ap.nb = nb;
    ap.tilesA = ntiles * (ntiles + 1) / 2;
    ap.tilesV = ntiles * ntiles;
    CUtensorMap mAh, mAl, mVh, mVl, mJh, mJl;
    bool ok = tj_map(&mAh, Ah, D, D, nb, JW) && tj_map(&mAl, Al, D, D, nb, JW) && tj_map(&mVh, Vh, D, D, nb, JW) &&
              tj_map(&mVl, Vl, D, D, nb, JW) && tj_map(&mJh, JPh, JP, JP, nb * ntiles, JP) &&
              tj_map(&mJl, JPl, JP, JP, nb * ntiles, JP);
    if (!ok) {
        // tensor maps unavailable: report through every matrix's status (no silent fallback)
        tj_fill_status_kernel<<<(nb + 127) / 128, 128, 0, s>>>(status, nb, ASG_ERR_CUDA);
        return;
    }
    const int debug = getenv("ASG_EIGH_DEBUG") != nullptr ? 1 : 0;
    const float ftol = float(tol);
    const int inner = getenv("ASG_TJ_INNER") ? atoi(getenv("ASG_TJ_INNER")) : kInner;
    static const int oe_env = getenv("ASG_TJ_OE") ? atoi(getenv("ASG_TJ_OE")) : -1;  // tuning override
    const int oe = oe_env >= 0 ? oe_env : (wide ? kOddEvenWide : kOddEvenNarrow);
    static const int rot32 = getenv("ASG_TJ_ROT32") ? atoi(getenv("ASG_TJ_ROT32")) : kRot32;  // tuning
    static const int nt_wide = getenv("ASG_TJ_NT") ? atoi(getenv("ASG_TJ_NT")) : 512;      // tuning
    const int total_tiles = nb * (ap.tilesA + ap.tilesV);
    const int apply_grid = total_tiles < num_sms ? total_tiles : num_sms;

    int* big = rotations;  // per-matrix "some element still above threshold" (tj_check_kernel)
    auto check = [&](cudaStream_t st, int count_sweep) {
        tj_check_kernel<<<dim3(D / 32, nb), 256, size_t(D) * 4, st>>>(Ah, Al, D, n, fro, active, big, ftol);
        tj_settle_kernel<<<(nb + 127) / 128, 128, 0, st>>>(nb, active, big, sweeps, debug, n, count_sweep);
    };
    auto prologue = [&](cudaStream_t st) {
        cudaMemsetAsync(sweeps, 0, size_t(nb) * 2 * sizeof(int), st);  // sweeps, rotations/big
        cudaMemsetAsync(loop_count, 0, sizeof(int), st);
        // J tiles: the pair kernels write their diagonal PW x PW blocks only
        cudaMemsetAsync(JPh, 0, size_t(nb) * ntiles * JP * JP * 2 * sizeof(float), st);
        unsigned* bound_bits = reinterpret_cast<unsigned*>(rank);  // rank[] is free until the epilogue
        int* bad = rank + nb;
        cudaMemsetAsync(fro, 0, size_t(nb) * sizeof(double), st);
        cudaMemsetAsync(rank, 0, size_t(nb) * 2 * sizeof(int), st);
        tj_stats_kernel<<<dim3(D / 32, nb), 256, 0, st>>>(B, n, D, fro, bound_bits, bad);
        tj_stats_finish_kernel<<<(nb + 127) / 128, 128, 0, st>>>(nb, fro, pad, bound_bits, bad, active, status);
        tj_init_kernel<<<dim3(D / 32, D / 32, nb), dim3(32, 8), 0, st>>>(B, n, D, pad, Ah, Al, Vh, Vl);
        check(st, 0);  // already diagonal to the threshold (warm refresh): no sweep at all
    };
    auto sweep = [&](cudaStream_t st) {
        for (int r = 0; r < m - 1; ++r) {
            TJApply a = ap;
            a.round = r;
            if (wide) {
                if (nt_wide == 1024)
                    tj_pair_kernel<128, 1024><<<dim3(npairs, nb), 1024, 2 * 128 * 129 * 4, st>>>(
                        Ah, Al, D, m, r, JPh, JPl, pflag, rotations, active, fro, n, ftol, inner, oe, rot32);
                else
                    tj_pair_kernel<128, 512><<<dim3(npairs, nb), 512, 2 * 128 * 129 * 4, st>>>(
                        Ah, Al, D, m, r, JPh, JPl, pflag, rotations, active, fro, n, ftol, inner, oe, rot32);
                tj_apply_kernel<64><<<apply_grid, 192, kApplySmem, st>>>(mAh, mAl, mVh, mVl, mJh, mJl, a);
            } else {
                tj_pair_kernel<64, 256><<<dim3(npairs, nb), 256, 2 * 64 * 65 * 4, st>>>(
                    Ah, Al, D, m, r, JPh, JPl, pflag, rotations, active, fro, n, ftol, inner, oe, rot32);
                tj_apply_kernel<32><<<apply_grid, 192, kApplySmem, st>>>(mAh, mAl, mVh, mVl, mJh, mJl, a);
            }
        }
        check(st, 1);
    };
    auto epilogue = [&](cudaStream_t st) {
        tj_rank_kernel<<<nb, 512, size_t(D) * 4, st>>>(Ah, Al, n, D, rank, values, active, status, sweeps, ident);
        tj_gather_kernel<<<dim3(256, nb), 256, 0, st>>>(Vh, Vl, rank, n, D, Jh, Jl);
        launch_transpose_split(Jh, Jl, nb, D, D, JTh, JTl, false, st);
    };
    // W = B J (3xTF32, or TF32 when the outputs carry no lo part), then
    // Rayleigh quotients + unit columns. Enqueued outside the cached graph.
    auto rayleigh = [&](cudaStream_t st) {
        launch_split_slab(B, Ah, Al, int64_t(size_t(nb) * DD), st);
        GemmLaunch gl{};
        gl.A = Operand{Ah, Al, D, D};
        gl.B = Operand{JTh, JTl, D, D};
        gl.batch = nb;
        gl.epi = EPI_STORE;
        gl.p.alpha = 1.f;
        gl.p.beta = 0.f;
        gl.p.C = Vh;
        gl.p.ldc = D;
        gl.p.c_bstride = int64_t(DD);
        gl.p.batch_active = sweeps;  // unswept matrices (J a permutation) need no W
        gemm_launch(gl, JTl ? ASG_PREC_3XTF32 : ASG_PREC_TF32, num_sms, st);
        tj_rayleigh_kernel<<<dim3(D / 32, nb), 256, 0, st>>>(Jh, Jl, JTh, JTl, Vh, n, D, values, B, D, sweeps);
        tj_sort_values_kernel<<<nb, 512, size_t(n) * 8, st>>>(values, n);
        count_launch(2);  // rayleigh + sort (split / GEMM count themselves)
        if (!orthonormalize) return;
        // one Newton-Schulz polar step on J (orthonormal to the fp32 floor):
        // S = J^T J -> X = (3I - S)/2 -> J X; A/V slabs are free scratch here
        GemmLaunch gs{};
        gs.A = Operand{JTh, JTl, D, D};
        gs.B = Operand{JTh, JTl, D, D};
        gs.batch = nb;
        gs.epi = EPI_STORE;
        gs.p.alpha = 1.f;
        gs.p.beta = 0.f;
        gs.p.C = Vh;
        gs.p.ldc = D;
        gs.p.c_bstride = int64_t(DD);
        gemm_launch(gs, JTl ? ASG_PREC_3XTF32 : ASG_PREC_TF32, num_sms, st);
        launch_ns_x(Vh, nb, n, D, Vh, JTl ? Vl : nullptr, st);
        GemmLaunch gx{};
        gx.A = Operand{Jh, Jl, D, D};
        gx.B = Operand{Vh, JTl ? Vl : nullptr, D, D};
        gx.batch = nb;
        gx.epi = EPI_SPLIT;
        gx.p.alpha = 1.f;
        gx.p.Dhi = Ah;
        gx.p.Dlo = JTl ? Al : nullptr;
        gx.p.ldd = D;
        gx.p.d_bstride = int64_t(DD);
        gemm_launch(gx, JTl ? ASG_PREC_3XTF32 : ASG_PREC_TF32, num_sms, st);
        cudaMemcpyAsync(Jh, Ah, size_t(nb) * DD * 4, cudaMemcpyDeviceToDevice, st);
        if (Jl) cudaMemcpyAsync(Jl, Al, size_t(nb) * DD * 4, cudaMemcpyDeviceToDevice, st);
        launch_transpose_split(Ah, Jl ? Al : nullptr, nb, D, D, JTh, JTl, false, st);
    };
    if (debug) {
        prologue(s);
        for (int k = 0; k < kEighMaxLaunchedSweeps; ++k) sweep(s);
        epilogue(s);
        rayleigh(s);
        count_launch(4 + uint64_t(kEighMaxLaunchedSweeps) * (2 * uint64_t(m - 1) + 1));
        return;
    }
    static std::mutex mu;
    using Key = std::tuple<const void*, const void*, const void*, const void*, const void*, const void*, const void*,
                           const void*, int, int, float, int, const void*>;
    static std::map<Key, cudaGraphExec_t> cache;
    const Key key{B, values, Jh, Jl, JTh, JTl, ws, status, nb, n, ftol, inner, ident};
    cudaGraphExec_t exec = nullptr;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) exec = it->second;
    }
    if (!exec) {
        cudaStream_t cap;
        cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
        auto capture = [&](auto&& body) {
            cudaGraph_t gph = nullptr;
            cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
            body(cap);
            cudaStreamEndCapture(cap, &gph);
            return gph;
        };
        cudaGraph_t g = nullptr;
        cudaGraphCreate(&g, 0);
        cudaGraphConditionalHandle handle;
        cudaGraphConditionalHandleCreate(&handle, g, 0, cudaGraphCondAssignDefault);
        cudaGraph_t gpro = capture(prologue);
        cudaGraph_t gepi = capture(epilogue);
        cudaGraphNode_t npro, ndecide, nloop, nepi;
        cudaGraphAddChildGraphNode(&npro, g, nullptr, 0, gpro);
        // enter the loop only if the prologue's check left a matrix active
        int max_sweeps = kEighMaxLaunchedSweeps;
        void* kargs[] = {&active, &nb, &loop_count, &max_sweeps, &handle};
        cudaKernelNodeParams kp{};
        kp.func = reinterpret_cast<void*>(tj_loop_kernel);
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(256);
        kp.sharedMemBytes = 0;
        kp.kernelParams = kargs;
        cudaGraphAddKernelNode(&ndecide, g, &npro, 1, &kp);
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = handle;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphAddNode(&nloop, g, &ndecide, 1, &cp);
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        sweep(cap);
        tj_loop_kernel<<<1, 256, 0, cap>>>(active, nb, loop_count, kEighMaxLaunchedSweeps, handle);
        cudaStreamEndCapture(cap, &body);
        cudaGraphAddChildGraphNode(&nepi, g, &nloop, 1, gepi);
        cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(gpro);
        cudaGraphDestroy(gepi);
        cudaGraphDestroy(g);
        cudaStreamDestroy(cap);
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = exec;
    }
    count_launch(4 + 2 * uint64_t(m - 1) + 2 + 2);
    cudaGraphLaunch(exec, s);
    static const bool report = getenv("ASG_TJ_REPORT") != nullptr;  // diagnostics: sweeps per solve
    if (report) {
        std::vector<int> sw;
        sw.resize(size_t(nb));
        int loops = 0;
        cudaMemcpyAsync(sw.data(), sweeps, size_t(nb) * sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&loops, loop_count, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        int mx = 0, mn = 1 << 30;
        for (int v : sw) {
            mx = v > mx ? v : mx;
            mn = v < mn ? v : mn;
        }
        fprintf(stderr, "tjreport n=%d nb=%d loops=%d sweeps min=%d max=%d\n", n, nb, loops, mn, mx);
    }
    rayleigh(s);
}
}  // namespace

void launch_tc_eigh(const float* B, int D_in, double* values, float* Jh, float* Jl, float* JTh, float* JTl, float* ws,
                    int nb, int n, int* status, int num_sms, cudaStream_t s, double tol, bool orthonormalize,
                    int* ident) {
    // the apply kernel keeps every pair flag of a launch in shared memory
    const int D = (n + JP - 1) / JP * JP;
    static const int wide_n = getenv("ASG_TJ_WIDE_N") ? atoi(getenv("ASG_TJ_WIDE_N")) : kWidePairN;
    const int npairs = D / (n >= wide_n ? 64 : 32) / 2;
    const int sub = kMaxFlags / npairs;
    const size_t DD = size_t(D) * D;
    for (int b0 = 0; b0 < nb; b0 += sub) {
        const int cnt = nb - b0 < sub ? nb - b0 : sub;
        tc_eigh_chunk(B + size_t(b0) * DD, D_in, values + size_t(b0) * n, Jh + size_t(b0) * DD,
                      Jl ? Jl + size_t(b0) * DD : nullptr, JTh + size_t(b0) * DD, JTl ? JTl + size_t(b0) * DD : nullptr,
                      ws, cnt, n, status + b0, num_sms, s, tol, orthonormalize, ident ? ident + b0 : nullptr);
    }
}

}  // namespace asg
