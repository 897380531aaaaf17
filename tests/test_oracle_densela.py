# SPDX-License-Identifier: Apache-2.0
"""Pins the oracle's densela restatement against the reference's own
known-answer tests (proj/tests/densela_test.cpp) and against LAPACK.

Each test cites the reference test it replays.
"""
import numpy as np
import pytest
import scipy.linalg

import orc
from paper_2605_16184_b200 import abi


def residual(m, vals, vecs):
    return np.abs(vecs @ np.diag(vals) @ vecs.T - m).max()


def test_sym_eig_identity():  # densela_test.cpp:23-28
    vals, vecs = orc.sym_eig(np.eye(3))
    assert np.allclose(vals, 1.0, rtol=1e-14, atol=0)
    assert np.abs(vecs.T @ vecs - np.eye(3)).max() < 1e-12


def test_sym_eig_diagonal_analytic_ascending():  # densela_test.cpp:30-42
    vals, vecs = orc.sym_eig(np.diag([4.0, 1.0]))
    assert vals[0] == 1.0 and vals[1] == 4.0
    assert abs(vecs[1, 0]) == 1.0 and abs(vecs[0, 1]) == 1.0
    assert vecs[0, 0] == 0.0 and vecs[1, 1] == 0.0


def test_sym_eig_random_spd_reconstructs():  # densela_test.cpp:44-48
    m = orc.random_spd(16, 42)
    vals, vecs = orc.sym_eig(m)
    assert residual(m, vals, vecs) < 1e-10


@pytest.mark.parametrize("dim", [2, 3, 8, 33, 64, 256])
def test_sym_eig_reconstruction_across_dims(dim):  # densela_test.cpp:50-61
    m = orc.random_spd(dim, 100 + dim)
    vals, vecs = orc.sym_eig(m)
    scale = np.abs(m).max()
    assert residual(m, vals, vecs) < 1e-8 * dim * scale
    assert np.abs(vecs.T @ vecs - np.eye(dim)).max() < 1e-8
    assert np.all(np.diff(vals) >= 0)


@pytest.mark.parametrize("dim", [64, 256])
def test_sym_eig_matches_lapack(dim):
    """Beyond the reference's tests: eigenvalues agree with LAPACK dsyevd."""
    m = orc.random_spd(dim, 7000 + dim)
    vals, vecs = orc.sym_eig(m)
    ref = scipy.linalg.eigh(m, eigvals_only=True)
    assert np.abs(vals - ref).max() < 1e-12 * np.abs(ref).max() * dim
    # Eigenvectors up to sign: |Q^T Q_lapack| = I for a simple spectrum.
    _, q_ref = scipy.linalg.eigh(m)
    assert np.abs(np.abs(vecs.T @ q_ref) - np.eye(dim)).max() < 1e-7


def test_sym_eig_rejects_non_finite():  # densela_test.cpp:63-67
    m = np.eye(2)
    m[0, 1] = m[1, 0] = np.nan
    with pytest.raises(abi.NonFiniteError):
        orc.sym_eig(m)


def test_inv_root_identity_and_diagonal():  # densela_test.cpp:69-80
    r = orc.inv_root(np.eye(4), 4, 0.0)
    assert np.abs(r - np.eye(4)).max() < 1e-14
    rd = orc.inv_root(np.diag([16.0, 1.0]), 4, 0.0)
    assert rd[0, 0] == pytest.approx(0.5, rel=1e-14)
    assert rd[1, 1] == pytest.approx(1.0, rel=1e-14)
    assert abs(rd[0, 1]) < 1e-15


def test_inv_root_extended_precision_and_operator_identity():  # densela_test.cpp:82-93
    m = orc.random_spd(32, 7)
    eps = 1e-8
    r = orc.inv_root(m, 4, eps)
    oracle = orc.inv_root_xp(m, 4, eps)
    assert np.abs(r - oracle).max() < 1e-8
    damped = m + eps * np.eye(32)
    p4 = r @ r @ r @ r
    assert np.abs(p4 @ damped - np.eye(32)).max() < 1e-6


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("dim", [2, 8, 31, 64])
def test_inv_root_operator_identity(p, dim):  # densela_test.cpp:95-108
    m = orc.random_spd(dim, 900 + dim * 10 + p)
    eps = 1e-10
    r = orc.inv_root(m, p, eps)
    acc = np.eye(dim)
    for _ in range(p):
        acc = acc @ r
    assert np.abs(acc @ (m + eps * np.eye(dim)) - np.eye(dim)).max() < 1e-6 * dim


def test_inv_root_rejects_indefinite():  # densela_test.cpp:110-115
    with pytest.raises(abi.NotPsdError):
        orc.inv_root(np.diag([1.0, -2.0]), 4, 0.0)


def test_pack_unpack_bit_exact():  # densela_test.cpp:117-136
    one = np.array([[0.123456789]])
    p1 = orc.pack_spd(one)
    assert p1.size == 1 and p1[0] == 0.123456789
    m = orc.random_spd(3, 5)
    p = orc.pack_spd(m)
    assert p.size == 6
    assert orc.unpack_spd(p, 3).tobytes() == m.tobytes()
    for dim in (2, 7, 16, 65):
        s = orc.random_spd(dim, 300 + dim)
        assert orc.unpack_spd(orc.pack_spd(s), dim).tobytes() == s.tobytes()


def test_packed_storage_arithmetic():  # densela_test.cpp:138-145
    dim = 2048.0
    saved = dim * (dim - 1.0) / 2.0
    assert saved / (dim * dim) == pytest.approx(0.4998, rel=1e-3)
    assert dim * (dim + 1.0) / 2.0 + saved == dim * dim


def test_gram_contracts():  # densela_test.cpp:155-170
    row = orc.random_matrix(1, 5, 8)
    gl = orc.gram_left(row)
    assert gl.shape == (1, 1)
    assert gl[0, 0] == pytest.approx((row ** 2).sum(), rel=1e-14)
    assert np.abs(orc.gram_right(np.eye(3)) - np.eye(3)).max() == 0.0


def test_gram_outputs_psd():  # densela_test.cpp:172-185
    g = orc.random_matrix(4, 7, 11)
    vals, _ = orc.sym_eig(orc.gram_left(g))
    assert vals[0] >= -1e-12
    for s in range(8):
        x = orc.random_matrix(6, 9, 1000 + s)
        for m in (orc.gram_left(x), orc.gram_right(x)):
            vals, _ = orc.sym_eig(m)
            assert vals[0] >= -1e-10 * np.trace(m)


def test_random_matrix_is_libstdcxx_normal_stream():
    """The generator is std::mt19937_64 + std::normal_distribution
    (test_util.hpp:10-17): deterministic per seed, N(0,1) moments."""
    a = orc.random_matrix(200, 200, 1)
    b = orc.random_matrix(200, 200, 1)
    assert a.tobytes() == b.tobytes()
    assert abs(a.mean()) < 0.02 and abs(a.std() - 1.0) < 0.02


def test_checksum_is_fnv1a64():  # bytes.hpp:14-22
    # FNV-1a of the 8 bytes of 0.0 from the offset basis.
    h = 0xcbf29ce484222325
    for _ in range(8):
        h ^= 0
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    assert orc.checksum(np.zeros(1)) == h
