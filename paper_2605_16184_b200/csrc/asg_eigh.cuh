// SPDX-License-Identifier: Apache-2.0
//
// Batched symmetric eigensolver of the refresh (see asg_eigh.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace asg {

// At or below this dimension the direct parallel-Jacobi kernel (one CTA per
// matrix) is used; above it the batched block-Jacobi solver.
constexpr int kSmallEighN = 64;
// Sweeps enqueued per solve (converged matrices skip work device-side; the
// reference's budget is 30, densela.hpp:194). Non-convergence -> status.
constexpr int kEighMaxLaunchedSweeps = 30;

// fp64 workspace needed by launch_eigh for nb matrices of dimension n
// (cold start; `_warm` when an initial basis is passed).
size_t eigh_workspace_doubles(int nb, int n);
size_t eigh_workspace_doubles_warm(int nb, int n);
// A: [nb][n][n] fp64 symmetric (not modified). values: [nb][n] ascending.
// vectors: [nb][n][n], eigenvectors as columns. status: per-matrix asg_status
// (must be zero-initialised; only failures are written). Vinit (optional,
// [nb][n][n] orthogonal): warm start from a previous eigenbasis — the solve
// iterates on Vinit^T A Vinit, which is nearly diagonal when A changed little.
// Stopping rule: relative = 0 is the reference's off(A) <= 1e-12 ||A||_F
// (densela.hpp:192-203); relative = 1 rotates only elements with
// |a_ij| > tol * sqrt(a_ii a_jj), skips pairs without one, and stops after a
// sweep that rotated nothing (the fp32-level refresh).
struct EighOpts {
    int relative = 0;
    double tol = 0.0;
};
void launch_eigh(const double* A, double* values, double* vectors, double* ws, int nb, int n, int* status,
                 cudaStream_t s, const double* Vinit = nullptr, EighOpts opts = EighOpts{});

// Tensor-core block Jacobi of the F32 refresh (asg_jacobi_tc.cu).
// B: [nb][D][D] fp32 symmetric (leading n x n), D = tc_eigh_dim(n) (n > kSmallEighN).
// values: [nb][n] ascending (fp64). J / J^T: [nb][D][D] split tf32 pairs of the
// eigenvectors (columns of J), zero outside the leading n x n. ws: floats from
// tc_eigh_workspace_floats. status: per-matrix asg_status (zero-initialised).
int tc_eigh_dim(int n);
size_t tc_eigh_workspace_floats(int nb, int n);
// orthonormalize: one Newton-Schulz step on J (callers that re-orthonormalize
// the product Q J themselves pass false).
void launch_tc_eigh(const float* B, int D, double* values, float* Jh, float* Jl, float* JTh, float* JTl, float* ws,
                    int nb, int n, int* status, int num_sms, cudaStream_t s, double tol, bool orthonormalize = true,
                    int* ident = nullptr);  // optional per matrix: 1 if J is exactly the identity

// Coupled Newton-Schulz inverse p-th root (asg_newton.cu), p in {2, 4}:
// out = (A + eps_b I)^(-1/p) for the nb fp32 matrices A [nb][D][D] (leading
// d x d; out zero-padded, split pair). ws: ns_workspace_floats(nb, D) floats.
// status: per-matrix asg_status, failures only. sym_tiles: the D x D
// lower-triangle tile list (gemm_sym_tile_list).
size_t ns_workspace_floats(int nb, int D);
void launch_ns_inv_root(const float* A, int nb, int d, int D, const double* eps, int p, float* outh, float* outl,
                        float* ws, int* status, const int2* sym_tiles, int nsym, int precision, int num_sms,
                        cudaStream_t s);

}  // namespace asg
