# SPDX-License-Identifier: Apache-2.0
"""The batched C-ABI solvers (asg_inv_root_batched_f32: the NEWTON inverse
roots; asg_sym_eig_batched_f32: the F32 tensor-core Jacobi) against LAPACK,
in both NEWTON iterate arithmetics, and processed in chunks of the solvers'
scratch arena (ASG_BATCHED_SCRATCH_BYTES forces one matrix per chunk in a
subprocess): chunking changes neither result beyond the stated bounds.

Stated bounds (normwise relative): roots (A + eps I)^(-1/p), eps = damping
tr(A)/n, within 2e-5 s(n) of the fp64 eigendecomposition's, s(n) =
max(1, sqrt(n/384)) (tests/test_gpu_parity_large.py), for factors of condition
<= ~1e3 (the i^-2 spectrum is floored at 1e-3; at 1e4 both iterate
arithmetics reach 2-4.5e-5 for p = 2, the fp32 rounding of A amplified by the
root's conditioning); eigenpairs as tests/test_gpu_kernels.py (residual
2e-5 lambda_max)."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def spd_batch(n, batch, seed):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(batch):
        x = rng.standard_normal((n, 2 * n))
        a = x @ x.T / (2 * n) + 1e-3 * np.eye(n)
        if k == batch - 1:  # an LLM-like spectrum lambda_i ~ i^-2
            q = np.linalg.qr(rng.standard_normal((n, n)))[0]
            a = (q * (1.0 / np.arange(1, n + 1) ** 2 + 1e-3)) @ q.T
        out.append(a)
    return np.stack(out).astype(np.float32)


def ref_root(a, p, damping):
    a = a.astype(np.float64)
    eps = damping * np.trace(a) / a.shape[0]
    w, v = np.linalg.eigh(a + eps * np.eye(a.shape[0]))
    return (v * w ** (-1.0 / p)) @ v.T


def root_tol(n):
    return 2e-5 * max(1.0, np.sqrt(n / 384.0))


def run_inv_root(mats, p, damping, precision):
    from paper_2605_16184_b200 import runtime as rt
    a = torch.from_numpy(mats).cuda()
    out = torch.empty_like(a)
    rt.check(rt.lib.asg_inv_root_batched_f32(_ptr(a), _ptr(out), a.shape[0], a.shape[1], p, damping, precision, None))
    return out.cpu().numpy().astype(np.float64)


@pytest.fixture(scope="module")
def rt():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_16184_b200 import runtime
    assert runtime.device_supported(0)
    return runtime


@pytest.mark.parametrize("precision", [0, 3], ids=["3xtf32", "3xf16"])
@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("n", [200, 256, 520])
def test_inv_root_batched_matches_lapack(rt, n, p, precision):
    mats = spd_batch(n, 4, 10 + n + p)
    got = run_inv_root(mats, p, 1e-6, precision)
    for k in range(mats.shape[0]):
        ref = ref_root(mats[k], p, 1e-6)
        err = np.abs(got[k] - ref).max() / np.abs(ref).max()
        assert err <= root_tol(n), (k, err)


_CHUNKED = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import test_gpu_batched_solvers as T
import torch
from paper_2605_16184_b200 import runtime as rt
n = 256
mats = T.spd_batch(n, 5, 3)
for prec in (0, 3):
    got = T.run_inv_root(mats, 2, 1e-6, prec)
    np.save(%r + "/inv_%%d.npy" %% prec, got)
a = torch.from_numpy(mats).cuda()
vals = torch.empty(5, n, dtype=torch.float64, device="cuda")
vecs = torch.empty(5, n, n, dtype=torch.float32, device="cuda")
rt.check(rt.lib.asg_sym_eig_batched_f32(T._ptr(a), T._ptr(vals), T._ptr(vecs), 5, n, None))
np.save(%r + "/vals.npy", vals.cpu().numpy())
np.save(%r + "/vecs.npy", vecs.cpu().numpy())
print("OK")
"""


def test_chunked_batches_match_one_chunk(rt, tmp_path):
    """One matrix per chunk (ASG_BATCHED_SCRATCH_BYTES=1) against LAPACK and
    against the single-chunk roots."""
    code = _CHUNKED % (os.path.join(ROOT, "tests"), str(tmp_path), str(tmp_path), str(tmp_path))
    env = dict(os.environ, ASG_BATCHED_SCRATCH_BYTES="1",
               PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stderr[-3000:]
    mats = spd_batch(256, 5, 3)
    for prec in (0, 3):
        chunked = np.load(tmp_path / f"inv_{prec}.npy")
        whole = run_inv_root(mats, 2, 1e-6, prec)
        for k in range(5):
            ref = ref_root(mats[k], 2, 1e-6)
            assert np.abs(chunked[k] - ref).max() / np.abs(ref).max() <= root_tol(256)
            assert np.abs(chunked[k] - whole[k]).max() / np.abs(whole[k]).max() <= 1e-6
    vals, vecs = np.load(tmp_path / "vals.npy"), np.load(tmp_path / "vecs.npy").astype(np.float64)
    for k in range(5):
        a = mats[k].astype(np.float64)
        lam = np.abs(np.linalg.eigvalsh(a)).max()
        assert np.abs(a @ vecs[k] - vecs[k] * vals[k]).max() <= 2e-5 * lam
        assert np.abs(vecs[k].T @ vecs[k] - np.eye(256)).max() <= 2e-5
