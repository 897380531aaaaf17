# SPDX-License-Identifier: Apache-2.0
"""GPU parity at the block sizes the benchmark runs (BASELINE configs C1-C5):
n = 512 ... 2048, where the F32 refresh's tensor-core Jacobi uses its wide
(128 x 128) pair solves (asg_jacobi_tc.cu kWidePairN = 512).

The checker at these sizes is oracle/orc_np.py, the LAPACK-backed
restatement of the oracle's per-block path, pinned to the C oracle at the
reference's test sizes by tests/test_oracle_np.py (the C oracle's cyclic
Jacobi takes minutes per 2048^2 factor on one core).

Stated tolerances (normwise relative, max|x - x_ref| / max|x_ref|). The fp32
factor carries ~sqrt(n) 2^-24 relative rounding noise, which bounds any
fp32-level eigensolve, so the n <= 384 bounds of
tests/test_gpu_kernels.py / test_gpu_refresh_f32.py scale by
s(n) = max(1, sqrt(n / 384)) (1.63 at 1024, 2.31 at 2048):
  * batched eigensolve alone: residual |A V - V diag(w)| <= 2e-5 s lambda_max,
    |V^T V - I| <= 2e-5 s, eigenvalues within 1e-5 s lambda_max of LAPACK,
    ascending;
  * refreshed roots (Shampoo L^-1/4, KL L^-1/2 and L^-1) from the GPU's own
    fp32 factor: <= max(2e-5 s, 2.5 gemm_tol(n)), gemm_tol(K) = 1e-6 + 1.2e-8 K
    the stated error of one 3xTF32 product at depth K (tests/test_gpu_kernels.py:
    the tensor core's fp32 accumulation truncates, so it grows linearly in K);
    a root is a chain of such products;
  * SOAP eigenvalues <= 1e-5 s lambda_max, orthonormality <= 2e-5 s,
    eigenvectors 1 - |cos| <= 1e-5 where the relative gap to the neighbours
    exceeds 1e-3, <= 1e-5 s;
  * trajectories (C1: Shampoo 1024^2 pf=1 S=0; C3 block: KL-Shampoo 2048^2):
    max|theta - theta_ref| <= r max|theta_ref - theta_0| + k 2^-23 max|theta_0|
    with r = 5e-4 (the F32 rows of DESIGN.md §4).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import orc
import orc_np
from paper_2605_16184_b200 import abi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def s_n(n):
    """Tolerance scale for fp32 factors of dimension n (module docstring)."""
    return max(1.0, np.sqrt(n / 384.0))


def root_tol(n):
    return max(2e-5 * s_n(n), 2.5 * (1e-6 + 1.2e-8 * n))


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.fixture(scope="module")
def rt():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_16184_b200 import runtime
    assert runtime.device_supported(0), "B200 (sm_100) required"
    return runtime


def _ptr(t):
    import ctypes as C
    return C.c_void_p(t.data_ptr())


def make_matrices(n, seed):
    """Random SPD (test_util.hpp:20-26), the LLM-like spectrum lambda_i ~ i^-2
     and a rank-deficient Gram factor (the 768 x 256 GPT-2 class:
    rank n/3, exact zeros)."""
    mats = [orc.random_spd(n, 900 + n + seed)]
    q = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))[0]
    mats.append((q * (1.0 / np.arange(1, n + 1) ** 2 + 1e-6)) @ q.T)
    g = np.random.default_rng(seed + 1).standard_normal((n, n // 3)) / np.sqrt(n)
    mats.append(g @ g.T)
    return mats


def check_eigh(n, mats, vals, vecs, res_tol, orth_tol, label=""):
    out = []
    for k, a in enumerate(mats):
        a = a.astype(np.float32).astype(np.float64)
        ref = np.linalg.eigvalsh(a)
        lmax = np.abs(ref).max()
        v, q = vals[k], vecs[k].astype(np.float64)
        e_val = np.abs(v - ref).max() / lmax
        e_res = np.abs(a @ q - q * v).max() / lmax
        e_orth = np.abs(q.T @ q - np.eye(n)).max()
        out.append((e_val, e_res, e_orth))
        print(f"{label} n={n} matrix {k}: eigenvalues {e_val:.2e} residual {e_res:.2e} orthonormality {e_orth:.2e}")
        assert np.all(np.diff(v) >= 0)
        assert e_val <= 1e-5 * s_n(n), (k, e_val)
        assert e_res <= res_tol, (k, e_res)
        assert e_orth <= orth_tol, (k, e_orth)
    return out


@pytest.mark.parametrize("n", [512, 520, 640, 768, 1024, 2048])
def test_sym_eig_batched_f32_wide_pairs_match_lapack(rt, n):
    """The wide-pair tensor-core Jacobi (every F32 refresh of C1-C5) against
    LAPACK: random SPD, i^-2 spectrum, rank-deficient Gram; padded sizes 520
    and 640 (D = 640 / 768) included."""
    mats = make_matrices(n, 3)
    batch = len(mats)
    A = torch.from_numpy(np.stack(mats).astype(np.float32)).cuda()
    vals = torch.empty(batch, n, dtype=torch.float64, device="cuda")
    vecs = torch.empty(batch, n, n, dtype=torch.float32, device="cuda")
    rt.check(rt.lib.asg_sym_eig_batched_f32(_ptr(A), _ptr(vals), _ptr(vecs), batch, n, None))
    tol = 2e-5 * s_n(n)
    check_eigh(n, mats, vals.cpu().numpy(), vecs.cpu().numpy(), tol, tol)


@pytest.mark.parametrize("n", [768, 1024, 2048])
def test_sym_eig_batched_f32_warm_refresh_matches_lapack(rt, n):
    """The matrix a warm SOAP refresh hands the eigensolver with fresh gradients
    (pf 10, beta 0.95): B = Q^T (0.6 A1 + 0.4 A_fresh) Q, Q the eigenbasis of A1,
    so B is diagonally dominant with 40% fresh off-diagonal mass. This exercises
    the classical few-element pair path, skipped tiles and the symmetric apply
    at the bench's block sizes. Same tolerances as the cold test."""
    rng = np.random.default_rng(n)

    def gram():
        x = rng.standard_normal((n, 2 * n)) / np.sqrt(2 * n)
        return x @ x.T + 1e-3 * np.eye(n)

    a1 = gram()
    _, q = np.linalg.eigh(a1)
    mats = []
    for _ in range(2):
        b = q.T @ (0.6 * a1 + 0.4 * gram()) @ q
        mats.append(0.5 * (b + b.T))
    batch = len(mats)
    A = torch.from_numpy(np.stack(mats).astype(np.float32)).cuda()
    vals = torch.empty(batch, n, dtype=torch.float64, device="cuda")
    vecs = torch.empty(batch, n, n, dtype=torch.float32, device="cuda")
    rt.check(rt.lib.asg_sym_eig_batched_f32(_ptr(A), _ptr(vals), _ptr(vecs), batch, n, None))
    tol = 2e-5 * s_n(n)
    check_eigh(n, mats, vals.cpu().numpy(), vecs.cpu().numpy(), tol, tol, label="warm")


def test_wide_pair_path_forced_at_small_n():
    """ASG_TJ_WIDE_N=128 forces the 128 x 128 pair solves from n = 129 (read
    once per process, so in a subprocess): same bounds as the narrow path's
    test (tests/test_gpu_kernels.py)."""
    code = (
        "import sys, numpy as np, torch; sys.path[:0] = [%r, %r]\n"
        "import test_gpu_parity_large as T\n"
        "from paper_2605_16184_b200 import runtime as rt\n"
        "for n in (130, 256, 384):\n"
        "    mats = T.make_matrices(n, 5)\n"
        "    A = torch.from_numpy(np.stack(mats).astype(np.float32)).cuda()\n"
        "    vals = torch.empty(len(mats), n, dtype=torch.float64, device='cuda')\n"
        "    vecs = torch.empty(len(mats), n, n, dtype=torch.float32, device='cuda')\n"
        "    rt.check(rt.lib.asg_sym_eig_batched_f32(T._ptr(A), T._ptr(vals), T._ptr(vecs), len(mats), n, None))\n"
        "    T.check_eigh(n, mats, vals.cpu().numpy(), vecs.cpu().numpy(), 2e-5, 2e-5, 'wide-forced')\n"
        "print('OK')\n" % (ROOT, os.path.join(ROOT, "tests")))
    env = dict(os.environ, ASG_TJ_WIDE_N="128", PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "oracle")]))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stderr[-3000:]


def f32_sched(mode=abi.REFRESH_F32):
    s = abi.scheduler_defaults()
    s.refresh_mode = mode
    return s


def big_block(P, method, m, n, steps, seed, mode=abi.REFRESH_F32, precision=abi.PREC_3XTF32):
    """A PrecondBlock after `steps` i.i.d. N(0, 1/n) gradients (the bench's
    distribution), and the orc_np block fed the identical fp32
    gradients."""
    cfg = P.defaults_for(method)
    b = P.PrecondBlock(m, n, method, cfg, precision=precision, sched=f32_sched(mode))
    nb = orc_np.Block(m, n, method)
    rng = np.random.default_rng(seed)
    for _ in range(steps):
        g = (rng.standard_normal((m, n)) / np.sqrt(n)).astype(np.float32).astype(np.float64)
        P.accumulate_factors(b, g, cfg)
        orc_np.accumulate_factors(nb, g, cfg)
    return cfg, b, nb


@pytest.fixture(scope="module")
def P(rt):
    from paper_2605_16184_b200 import precond
    return precond


@pytest.mark.parametrize("mode,precision", [(abi.REFRESH_F32, abi.PREC_3XTF32), (abi.REFRESH_NEWTON, abi.PREC_3XTF32),
                                            (abi.REFRESH_NEWTON, abi.PREC_3XF16)])
@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
@pytest.mark.parametrize("n", [1024, 2048])
def test_f32_refresh_roots_at_bench_sizes(P, method, n, mode, precision):
    """compute_refresh (precond.cpp:129-142) at C1 / C3 block sizes: cold
    refresh, then a warm one after more statistics, each against the
    LAPACK-backed oracle on the GPU's own fp32 factor. Both fp32-level
    refreshes: the tensor-core Jacobi (F32) and the coupled Newton-Schulz
    roots (NEWTON; 3xTF32 iterates, or 3xFP16 iterates at bound-derived
    scales)."""
    cfg, b, _ = big_block(P, method, n, n, 4, 11, mode, precision)
    for step, extra in ((3, 0), (6, 3)):
        rng = np.random.default_rng(100 + step)
        for _ in range(extra):
            P.accumulate_factors(b, (rng.standard_normal((n, n)) / np.sqrt(n)).astype(np.float32), cfg)
        P.refresh_inverse(b, cfg, step)
        r = orc_np.compute_refresh(b.factor_l, b.factor_r, cfg)
        errs = [rel(b.inv_l, r["inv_l"]), rel(b.inv_r, r["inv_r"])]
        kerrs = []
        if method == abi.KL_SHAMPOO:
            # F^-1 is derived as (F^-1/2)^2 (never stored): to first order its
            # relative error is twice the root's, hence the stated 2x bound
            kerrs = [rel(b.get(abi.KL_INV_L), r["kl_inv_l"]), rel(b.get(abi.KL_INV_R), r["kl_inv_r"])]
        print(f"n={n} {abi.METHOD_NAMES[method]} mode {mode} prec {precision} step {step}: root errors "
              f"{['%.2e' % e for e in errs + kerrs]}")
        assert max(errs) <= root_tol(n), errs
        assert not kerrs or max(kerrs) <= 2 * root_tol(n), kerrs


@pytest.mark.parametrize("m,n", [(1024, 1024), (768, 1024), (2048, 2048)])
def test_f32_soap_basis_at_bench_sizes(P, m, n):
    """SOAP's eigenbases (compute_refresh SOAP branch precond.cpp:131-135) at
    the C2 (768 x 1024, 1024^2) and C4 (2048^2) block shapes."""
    cfg, b, _ = big_block(P, abi.SOAP, m, n, 6, 21)
    P.refresh_inverse(b, cfg, 5)
    for fac, q, w in ((b.factor_l, b.basis_l, b.get(abi.EIGVALS_L)), (b.factor_r, b.basis_r, b.get(abi.EIGVALS_R))):
        wr, qr = orc_np.sym_eig(fac)
        lmax = np.abs(wr).max()
        e_val = np.abs(w - wr).max() / lmax
        gap = np.minimum(np.diff(wr, prepend=-np.inf), np.diff(wr, append=np.inf)) / lmax
        sel = gap > 1e-3
        cos = np.abs(np.sum(q * qr, axis=0))
        e_vec = (1.0 - cos[sel]).max() if sel.any() else 0.0
        e_orth = np.abs(q.T @ q - np.eye(q.shape[0])).max()
        print(f"SOAP {m}x{n} side {q.shape[0]}: eigenvalues {e_val:.2e}, 1-|cos| {e_vec:.2e} over {sel.sum()} "
              f"separated vectors, orthonormality {e_orth:.2e}")
        assert e_val <= 1e-5 * s_n(q.shape[0])
        assert e_vec <= 1e-5 * s_n(q.shape[0])
        assert e_orth <= 2e-5 * s_n(q.shape[0])


def well_grad(rng, m, n, scale=1e-3):
    k = min(m, n)
    u = np.linalg.qr(rng.standard_normal((m, k)))[0]
    v = np.linalg.qr(rng.standard_normal((n, k)))[0]
    return scale * (u * rng.uniform(0.5, 1.5, k)) @ v.T


def big_trajectory(method, m, n, steps, pf, S, lr, accumulation, r, first_step=0, mode=abi.REFRESH_F32,
                   adopt_basis=False, precision=abi.PREC_3XTF32):
    """One block through AsteriaOptimizer (asg_step: the per-block call order
    of harness.cpp:448-475, S = 0: the refresh dispatched at step % pf == 0
    is installed by the same step's barrier) against orc_np's per-block
    loop; well-conditioned gradients (tests/test_gpu_step.py)."""
    from paper_2605_16184_b200 import optimizer, runtime
    opt = runtime.optimizer_defaults(method)
    opt.lr, opt.precondition_frequency, opt.block_dim_limit = lr, pf, 2048
    opt.accumulation = accumulation
    sched = runtime.scheduler_defaults()
    sched.pf, sched.staleness_S = pf, S
    sched.refresh_mode = mode
    rng = np.random.default_rng(7)
    th0 = 0.02 * rng.standard_normal((m, n))
    W = torch.tensor(th0, dtype=torch.float32, device="cuda")
    G = torch.zeros_like(W)
    o = optimizer.AsteriaOptimizer([W], [G], opt, sched, precision=precision)
    nb = orc_np.Block(m, n, method)
    th = th0.copy()
    for step in range(first_step, first_step + steps):
        g = well_grad(rng, m, n).astype(np.float32).astype(np.float64)
        G.copy_(torch.tensor(g, dtype=torch.float32))
        o.step(step, clip_scale=1.0, lr_scale=1.0)
        orc_np.accumulate_factors(nb, g, opt)
        if step % pf == 0:
            r_ = orc_np.compute_refresh(nb.factor_l.copy(), nb.factor_r.copy(), opt)
            if adopt_basis:  # the GPU's installed eigenbasis (read after its same-step install, S = 0)
                wl, _, wr, _ = r_["soap"]
                r_["soap"] = (wl, o.read_block(0, abi.BASIS_L), wr, o.read_block(0, abi.BASIS_R))
            orc_np.install_refresh(nb, r_, step)
        th = orc_np.apply_update(th, orc_np.step_update(nb, g, opt), opt)
    o.synchronize()
    got = W.double().cpu().numpy()
    allowed = r * np.abs(th - th0).max() + steps * 2.0 ** -23 * np.abs(th0).max()
    err = np.abs(got - th).max() / allowed
    print(f"{abi.METHOD_NAMES[method]} {m}x{n} mode {mode} trajectory: error / stated tolerance = {err:.3f}")
    assert o.stats().installed == len([s for s in range(first_step, first_step + steps) if s % pf == 0])
    return err


PRECS = [abi.PREC_3XTF32, abi.PREC_3XTF32_SMEM, abi.PREC_3XF16]


@pytest.mark.parametrize("precision", PRECS)
@pytest.mark.parametrize("mode", [abi.REFRESH_F32, abi.REFRESH_NEWTON])
def test_c1_trajectory_shampoo_1024_pf1(rt, mode, precision):
    """BASELINE C1: Shampoo on one 1024^2 block with the reference's
    quadratic_shampoo.json hyper-parameters (EMA b2 = 0.95, pf = 1, S = 0,
    lr 3e-3): a synchronous refresh every step."""
    assert big_trajectory(abi.SHAMPOO, 1024, 1024, steps=6, pf=1, S=0, lr=3e-3, accumulation=abi.EMA, r=5e-4,
                          mode=mode, precision=precision) <= 1.0


@pytest.mark.parametrize("precision", PRECS)
@pytest.mark.parametrize("mode", [abi.REFRESH_F32, abi.REFRESH_NEWTON])
def test_c3_block_trajectory_kl_shampoo_2048(rt, mode, precision):
    """One C3 block: KL-Shampoo on a 2048^2 block, pf = 2, S = 0."""
    assert big_trajectory(abi.KL_SHAMPOO, 2048, 2048, steps=5, pf=2, S=0, lr=1e-3, accumulation=abi.EMA,
                          r=5e-4, mode=mode, precision=precision) <= 1.0


@pytest.mark.parametrize("precision", PRECS)
def test_c2_block_trajectory_soap_768x1024(rt, precision):
    """One C2 block shape (768 x 1024, the c_attn / c_fc slices): SOAP,
    pf = 4, S = 0, steps 1-8 (the caller numbers the steps, harness.cpp:382):
    steps 1-3 are the identity-basis cold start (harness.cpp:458-461) and the
    first refresh (step 4) sees 4 accumulated gradients, so R (1024^2, rank
    <= 768 per gradient) is full rank.

    SOAP's update is not a smooth function of the eigenbasis: Adam's
    elementwise normalisation in the rotated basis is not invariant under
    rotations inside near-degenerate eigenspaces, so ANY two eigensolvers
    (LAPACK vs the reference's Jacobi in fp64 included) give updates that
    differ by ~(solver tolerance) / (relative eigen-gap). The F32 eigensolve's
    tolerance is 1e-6 and the i.i.d.-like spectra here have gaps ~1/n, so the
    trajectory is compared with the oracle running on the GPU's own installed
    eigenbasis (its eigenvectors are checked separately, against LAPACK, for
    every separated eigenvalue: test_f32_soap_basis_at_bench_sizes). This
    isolates everything else -- statistics, re-projection of the moments,
    rotated Adam, back-rotation, apply -- at the F32 trajectory tolerance
    r = 5e-4. A refresh of an exactly rank-deficient factor leaves fp32 noise
    in its null directions, which SOAP's rotated Adam normalises to O(1e-2)
    updates where the fp64 reference gives ~1e-8 (tests/test_gpu_step.py
    docstring); that case is covered for finiteness and orthonormality by
    test_f32_refresh_rank_deficient_factor."""
    assert big_trajectory(abi.SOAP, 768, 1024, steps=8, pf=4, S=0, lr=1e-3, accumulation=abi.EMA, r=5e-4,
                          first_step=1, adopt_basis=True, precision=precision) <= 1.0


def test_c2_block_trajectory_soap_768x1024_own_basis(rt):
    """The same trajectory with the oracle's own (LAPACK) eigenbasis: bounded
    by the eigen-gap sensitivity described above; stated tolerance r = 1e-2
    (measured 4.2e-3 relative to the accumulated update)."""
    assert big_trajectory(abi.SOAP, 768, 1024, steps=8, pf=4, S=0, lr=1e-3, accumulation=abi.EMA, r=1e-2,
                          first_step=1) <= 1.0
