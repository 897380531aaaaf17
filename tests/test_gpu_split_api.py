# SPDX-License-Identifier: Apache-2.0
"""The reference's split refresh API and remaining per-block functions
through the C-ABI (precond.hpp:77-139): snapshot_factors / compute_refresh /
install_refresh, replicated_state / load_replicated_state, pack_spd /
unpack_spd, adamw_step / apply_update, replayed against the oracle and the
reference's own test cases (precond_test.cpp, densela_test.cpp)."""
import ctypes as C

import numpy as np
import pytest

import orc
from paper_2605_16184_b200 import abi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_16184_b200 import precond, runtime
    assert runtime.device_supported(0)
    return precond


def sched(mode):
    s = abi.scheduler_defaults()
    s.refresh_mode = mode
    return s


MODES = [abi.REFRESH_F64, abi.REFRESH_F32, abi.REFRESH_NEWTON]


@pytest.mark.parametrize("mode,precision", [(m, abi.PREC_3XTF32) for m in MODES] +
                         [(abi.REFRESH_NEWTON, abi.PREC_3XF16), (abi.REFRESH_F32, abi.PREC_3XF16)])
@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.SOAP, abi.KL_SHAMPOO])
def test_split_refresh_equals_refresh_inverse(P, method, mode, precision):
    """install(compute(snapshot)) is refresh_inverse (precond.cpp:166-171), also
    with 3XF16 step arithmetic (the install converts the roots to fp16 pairs)."""
    m, n = 96, 80
    cfg = P.defaults_for(method)
    a = P.PrecondBlock(m, n, method, cfg, precision=precision, sched=sched(mode))
    b = P.PrecondBlock(m, n, method, cfg, precision=precision, sched=sched(mode))
    for s in range(3):
        g = orc.random_matrix(m, n, 10 + s)
        P.accumulate_factors(a, g, cfg)
        P.accumulate_factors(b, g, cfg)
    P.refresh_inverse(a, cfg, 4)
    snap = P.snapshot_factors(b)
    P.install_refresh(b, P.compute_refresh(b, snap, cfg), 4)
    assert a.version == b.version == 1 and b.last_refresh_step == 4
    roles = ([abi.BASIS_L, abi.BASIS_R, abi.EIGVALS_L] if method == abi.SOAP else [abi.INV_L, abi.INV_R])
    for r in roles:
        x, y = a.get(r), b.get(r)
        if r in (abi.BASIS_L, abi.BASIS_R):  # compare the projectors column by column (sign-free)
            assert np.abs(np.abs(np.sum(x * y, axis=0)) - 1).max() < 1e-5
        else:
            assert rel(y, x) < 1e-6, r
    g = orc.random_matrix(m, n, 20)
    ua = P.precondition_soap(a, g, cfg) if method == abi.SOAP else P.precondition_shampoo(a, g)
    ub = P.precondition_soap(b, g, cfg) if method == abi.SOAP else P.precondition_shampoo(b, g)
    assert rel(ub, ua) < 1e-4


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
def test_snapshot_isolation(P, method, mode):
    """asyncsched_test.cpp:146-164: a refresh computed from a snapshot taken
    before further accumulation equals the oracle's refresh of the old
    factors; the snapshot's checksum does not change, the block's factors
    do."""
    m, n = 64, 48
    cfg = P.defaults_for(method)
    b = P.PrecondBlock(m, n, method, cfg, sched=sched(mode))
    for s in range(3):
        P.accumulate_factors(b, orc.random_matrix(m, n, 30 + s), cfg)
    old_l, old_r = b.factor_l, b.factor_r
    snap = P.snapshot_factors(b)
    c0 = snap.checksum
    for s in range(2):
        P.accumulate_factors(b, orc.random_matrix(m, n, 40 + s), cfg)
    assert snap.checksum == c0
    assert not np.array_equal(b.factor_l, old_l)
    res = P.compute_refresh(b, snap, cfg)
    assert b.version == 0  # compute_refresh is pure
    P.install_refresh(b, res, 7)
    o = orc.Block(m, n, method)
    o.set(abi.FACTOR_L, old_l)
    o.set(abi.FACTOR_R, old_r)
    orc.refresh_inverse(o, cfg, 7)
    assert rel(b.inv_l, o.inv_l) < 2e-5
    assert rel(b.inv_r, o.inv_r) < 2e-5
    snap2 = P.snapshot_factors(b)
    assert snap2.checksum != c0


@pytest.mark.parametrize("mode", MODES)
def test_soap_install_reprojects_permuted_basis(P, mode):
    """precond_test.cpp:139-164 through the split API: installing a basis that
    permutes the coordinates permutes the rotated moments."""
    cfg = P.defaults_for(abi.SOAP)
    cfg.damping = 0.0
    b = P.PrecondBlock(4, 4, abi.SOAP, cfg, sched=sched(mode))
    b.set(abi.FACTOR_L, np.diag([1.0, 2.0, 3.0, 4.0]))
    b.set(abi.FACTOR_R, np.eye(4))
    P.refresh_inverse(b, cfg, 0)
    mom = np.arange(16, dtype=float).reshape(4, 4) * 0.01
    b.set(abi.ROTATED_M, mom)
    b.set(abi.FACTOR_L, np.diag([4.0, 3.0, 2.0, 1.0]))
    snap = P.snapshot_factors(b)
    P.install_refresh(b, P.compute_refresh(b, snap, cfg), 1)
    got = b.rotated_m
    # eigenvalues ascending: the new basis reverses the coordinate order of L
    assert np.abs(np.abs(got) - np.abs(mom[::-1, :])).max() < 1e-6


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.SOAP])
def test_replicated_state_round_trip(P, method):
    """replicated_state / load_replicated_state (precond.cpp:253-279):
    [L side | R side] of the roots or bases; loading a state into a fresh
    block makes its preconditioning identical; a wrong size is ShapeMismatch."""
    m, n = 40, 24
    cfg = P.defaults_for(method)
    b = P.PrecondBlock(m, n, method, cfg, sched=sched(abi.REFRESH_F64))
    for s in range(3):
        P.accumulate_factors(b, orc.random_matrix(m, n, 50 + s), cfg)
    P.refresh_inverse(b, cfg, 2)
    flat = P.replicated_state(b)
    assert flat.shape == (m * m + n * n,)
    left = b.basis_l if method == abi.SOAP else b.inv_l
    assert np.array_equal(flat[:m * m].reshape(m, m), left)
    c = P.PrecondBlock(m, n, method, cfg, sched=sched(abi.REFRESH_F64))
    c.set_counters(1, 2, 0)
    P.load_replicated_state(c, flat)
    assert np.array_equal(P.replicated_state(c), flat)
    with pytest.raises(abi.ShapeMismatchError):
        P.load_replicated_state(c, flat[:-1])
    if method == abi.SHAMPOO:
        g = orc.random_matrix(m, n, 60)
        assert rel(P.precondition_shampoo(c, g), P.precondition_shampoo(b, g)) < 1e-6


def test_pack_unpack_spd_bit_exact(P):
    """densela_test.cpp:117-153: pack_spd / unpack_spd are bit-exact (fp32 on
    the device; the packed order is the reference's row-major lower
    triangle)."""
    from paper_2605_16184_b200 import runtime
    for n in (1, 2, 33, 130):
        mats = np.stack([orc.random_spd(n, 70 + n + k) for k in range(3)]).astype(np.float32)
        A = torch.from_numpy(mats).cuda()
        packed = torch.empty(3, n * (n + 1) // 2, dtype=torch.float32, device="cuda")
        back = torch.empty_like(A)
        runtime.check(runtime.lib.asg_pack_spd_f32(C.c_void_p(A.data_ptr()), 3, n, C.c_void_p(packed.data_ptr()), None))
        runtime.check(runtime.lib.asg_unpack_spd_f32(C.c_void_p(packed.data_ptr()), 3, n, C.c_void_p(back.data_ptr()),
                                                     None))
        torch.cuda.synchronize()
        for k in range(3):
            ref = orc.pack_spd(mats[k].astype(np.float64))
            assert np.array_equal(packed[k].cpu().numpy().astype(np.float64), ref)
        sym = 0.5 * (mats + mats.transpose(0, 2, 1))  # random_spd is symmetric to rounding
        assert np.array_equal(back.cpu().numpy(), np.tril(mats) + np.transpose(np.tril(mats, -1), (0, 2, 1)))
        assert np.abs(back.cpu().numpy() - sym).max() <= 1e-6 * np.abs(sym).max()


def test_adamw_step_and_apply_update_match_oracle(P):
    """precond_test.cpp:283-342 through the per-call entry points: AdamW
    directions over 5 steps (fp32 moments: <= 2e-5 relative -- the bias
    correction 1/(1 - beta2^t) ~ 1e3 scales the moments' fp32 rounding),
    apply_update exact in fp64, NonFinite before any state change."""
    cfg = P.defaults_for(abi.ADAMW)
    cfg.weight_decay = 0.01
    st, so = P.AdamState(3, 5), orc.AdamState(3, 5)
    for s in range(5):
        g = orc.random_matrix(3, 5, 80 + s)
        assert rel(P.adamw_step(st, g, cfg), orc.adamw_step(so, g, cfg)) < 2e-5
    theta = orc.random_matrix(3, 5, 90)
    u = orc.random_matrix(3, 5, 91)
    assert np.array_equal(P.apply_update(theta, u, cfg, 0.5), orc.apply_update(theta, u, cfg, 0.5))
    bad = u.copy()
    bad[1, 1] = np.nan
    with pytest.raises(abi.NonFiniteError):
        P.apply_update(theta, bad, cfg)
    with pytest.raises(abi.NonFiniteError):
        P.adamw_step(st, bad, cfg)
    # the failed call left the moments untouched: the next step still matches
    g = orc.random_matrix(3, 5, 95)
    assert rel(P.adamw_step(st, g, cfg), orc.adamw_step(so, g, cfg)) < 2e-5
