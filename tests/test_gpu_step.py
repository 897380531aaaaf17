# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the full optimizer step through the public API
(AsteriaOptimizer -> asg_step) with the CPU oracle:

  * trajectories: the per-block loop of harness.cpp:439-471 / the synchronous
    oracle reference_opt.cpp:91-107 (S = 0), multi-block parameters with
    ragged remainder blocks (several shape groups) plus a 1-D AdamW parameter;
  * schedule: the bounded-staleness state machine (asyncsched.cpp) on the
    simulated clock — identical dispatch/install/barrier events, freshness
    records and counters as the oracle for the reference's own Rig cases
    (asyncsched_test.cpp);
  * event-driven installs keep the consumed-snapshot age within (S+1)*pf.

Stated tolerance for theta after k steps (fp32 state, 3xTF32 products, fp64
refresh, against the fp64 reference):
    max|theta_k - theta_ref| <= r * max|theta_ref - theta_0| + k * 2^-23 * max|theta_0|
with r = 2e-4 (Shampoo, KL-Shampoo, AdamW) and r = 5e-4 (SOAP, whose Adam
normalisation in the rotated basis amplifies relative error in small-|Ghat|
components); the second term is fp32 storage rounding of theta itself. Inputs are
well-conditioned (full-rank factors with separated spectra): in exactly
rank-deficient factor directions fp32 rounding noise is not below the
fp64 reference's and SOAP's Adam normalisation amplifies it (see
test_gpu_precond.py); rank-deficient runs are checked for finiteness and
for the eigenvalue-clamp semantics only.
"""
import numpy as np
import pytest

import orc
from paper_2605_16184_b200 import abi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def O():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_16184_b200 import optimizer, runtime
    assert runtime.device_supported(0)
    return optimizer


def run_pair(O, method, shapes, limit, pf, steps, seed=0, S=0, lr=1e-2, wd=0.0, clip=1.0, well=True, delay=0.0,
             refresh_mode=abi.REFRESH_F64, r_scale=1.0, precision=abi.PREC_3XTF32, grad_scale=None):
    """GPU step vs the oracle's per-block harness loop (harness.cpp:439-475) with
    the oracle's ShadowScheduler on the same simulated clock."""
    from paper_2605_16184_b200 import runtime
    opt = runtime.optimizer_defaults(method)
    opt.lr, opt.weight_decay, opt.block_dim_limit, opt.precondition_frequency = lr, wd, limit, pf
    sched = runtime.scheduler_defaults()
    sched.pf, sched.staleness_S, sched.inject_job_delay_steps = pf, S, delay
    sched.refresh_mode = refresh_mode
    rng = np.random.default_rng(seed)
    thetas0 = [0.1 * rng.standard_normal(s) for s in shapes]
    params = [torch.tensor(t, dtype=torch.float32, device="cuda") for t in thetas0]
    grads = [torch.zeros_like(p) for p in params]
    o = O.AsteriaOptimizer(params, grads, opt, sched, precision=precision)
    osched = orc.Scheduler(opt, sched, seed=1)
    ref, all_blocks = [], []
    for t in thetas0:
        t2 = t if t.ndim == 2 else t[None, :]
        if t2.shape[0] == 1 or t2.shape[1] == 1:
            ref.append(("adam", orc.AdamState(*t2.shape), t2.copy()))
        else:
            blocks = []
            for r in range(0, t2.shape[0], limit):
                for c in range(0, t2.shape[1], limit):
                    r1, c1 = min(t2.shape[0], r + limit), min(t2.shape[1], c + limit)
                    b = orc.Block(r1 - r, c1 - c, method)
                    blocks.append((r, r1, c, c1, b, len(all_blocks)))
                    all_blocks.append(b)
            ref.append(("blocks", blocks, t2.copy()))

    def grad_for(s):
        if len(s) == 1 or not well:
            return 1e-3 * rng.standard_normal(s)
        g = np.empty(s)
        for r in range(0, s[0], limit):  # each block well conditioned
            for c in range(0, s[1], limit):
                m, n = min(s[0], r + limit) - r, min(s[1], c + limit) - c
                k = min(m, n)
                u = np.linalg.qr(rng.standard_normal((m, k)))[0]
                v = np.linalg.qr(rng.standard_normal((n, k)))[0]
                g[r:r + m, c:c + n] = 1e-3 * (u * rng.uniform(0.5, 1.5, k)) @ v.T
        return g

    for step in range(steps):
        gs = [grad_for(s) for s in shapes]
        if grad_scale is not None:
            gs = [g * grad_scale(step) for g in gs]
        for g, gt in zip(grads, gs):
            g.copy_(torch.tensor(gt, dtype=torch.float32))
        o.clock_advance(sched.step_compute_us)
        o.step(step, clip_scale=clip, lr_scale=1.0)
        osched.advance(sched.step_compute_us)
        for (kind, st, th), g in zip(ref, gs):
            g2 = clip * (g if g.ndim == 2 else g[None, :])
            if kind == "adam":
                th[:] = orc.apply_update(th, orc.adamw_step(st, g2, opt), opt)
                continue
            for (r, r1, c, c1, blk, bid) in st:
                gb = g2[r:r1, c:c1]
                orc.accumulate_factors(blk, gb, opt)
                osched.maybe_dispatch(blk, bid, step)
                osched.staleness_barrier(blk, bid, step)
                upd = orc.step_update(blk, gb, opt)  # cold-start rule harness.cpp:455-466
                th[r:r1, c:c1] = orc.apply_update(th[r:r1, c:c1], upd, opt)
        osched.step_end(all_blocks, list(range(len(all_blocks))), step)
    o.synchronize()
    errs = []
    for p, (kind, st, th), t0 in zip(params, ref, thetas0):
        got = p.double().cpu().numpy().reshape(th.shape)
        t0 = t0.reshape(th.shape)
        r = r_scale * (5e-4 if (method == abi.SOAP and kind == "blocks") else 2e-4)
        allowed = r * np.abs(th - t0).max() + steps * 2.0 ** -23 * np.abs(t0).max()
        errs.append(np.abs(got - th).max() / allowed)  # <= 1 passes
    return errs, o


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.SOAP, abi.KL_SHAMPOO])
def test_trajectory_matches_oracle_bounded_staleness(O, method):
    """Square well-conditioned blocks of three shape groups (incl. a padded
    72 -> 128 one) plus a 1-D AdamW parameter; refresh every pf=4 steps with a
    2-step job on the simulated clock and S=3, so steps 0-2 run the cold-start
    rule and later steps consume bases/roots of an older snapshot (Ghat is
    dense, which keeps SOAP's Adam normalisation well posed in fp32)."""
    shapes = [(256, 384), (300,), (96, 96), (72, 72)]
    errs, o = run_pair(O, method, shapes, limit=128, pf=4, steps=10, S=3, delay=2.0)
    assert o.num_blocks == 6 + 1 + 1 + 1
    assert o.stats().installed >= 2 * 8
    assert max(errs) <= 1.0, errs


@pytest.mark.parametrize("precision", [abi.PREC_3XF16, abi.PREC_3XTF32_SMEM])
@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.SOAP, abi.KL_SHAMPOO])
def test_trajectory_operand_storage_modes(O, method, precision):
    """The same bounded-staleness trajectories with the step's operands stored
    as scaled fp16 (hi, lo) pairs multiplied by kind::f16 (3XF16; SOAP runs its
    chain as 3XTF32_SMEM there) and as plain fp32 split in shared memory
    (3XTF32_SMEM): the 3xTF32 tolerances hold unchanged."""
    shapes = [(256, 384), (300,), (96, 96), (72, 72)]
    errs, o = run_pair(O, method, shapes, limit=128, pf=4, steps=10, S=3, delay=2.0, precision=precision)
    assert max(errs) <= 1.0, errs


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.KL_SHAMPOO])
def test_f16_gradient_scale_prediction_survives_magnitude_jumps(O, method):
    """3XF16 writes each step's G at the scale predicted from the block's previous
    max and rewrites the blocks whose prediction fails (launch_prep_grad_f16_pred):
    gradients jumping 1e3x up (overflow side) and 1e-4x down (precision side)
    between steps, and an all-zero gradient step, keep the 3xTF32 tolerances
    against the oracle."""
    seq = [1.0, 1e3, 1e-1, 0.0, 1e-4, 1.0, 30.0, 1e-2, 1.0]  # (0: an all-zero gradient step)
    shapes = [(256, 256), (96, 96)]
    errs, _ = run_pair(O, method, shapes, limit=128, pf=2, steps=len(seq), S=1, delay=1.0,
                       precision=abi.PREC_3XF16, grad_scale=lambda s: seq[s])
    assert max(errs) <= 1.0, errs


def test_trajectory_synchronous_weight_decay_and_clip(O):
    # S = 0: refresh every step, consumed the same step (reference_opt.cpp:96-99)
    errs, _ = run_pair(O, abi.SHAMPOO, [(160, 160)], limit=2048, pf=1, steps=4, wd=0.1, clip=0.5)
    assert max(errs) <= 1.0, errs


@pytest.mark.parametrize("method", [abi.SHAMPOO, abi.SOAP, abi.KL_SHAMPOO])
def test_rank_deficient_factors_stay_finite(O, method):
    """Non-square blocks make one factor exactly rank-deficient at step 0;
    fp32 eigenvalues at -(rounding level) are clamped to 0 (no spurious
    NotPsd, densela.hpp:274-278 semantics otherwise), updates stay finite."""
    _, o = run_pair(O, method, [(200, 300), (64, 96)], limit=128, pf=2, steps=4, well=False)
    for p in o.params:
        assert torch.isfinite(p).all()


def test_blocks_are_uniform_groups_and_owned(O):
    _, o = run_pair(O, abi.SOAP, [(256, 640), (768,)], limit=256, pf=1, steps=1)
    infos = [o.block_info(i) for i in range(o.num_blocks)]
    shapes = sorted({(i.spec.row_end - i.spec.row_begin, i.spec.col_end - i.spec.col_begin) for i in infos if not i.use_adamw})
    assert shapes == [(256, 128), (256, 256)]
    assert sum(i.use_adamw for i in infos) == 1
    assert all(i.owner_rank == 0 for i in infos)


# ---- schedule parity on the simulated clock (asyncsched_test.cpp Rig) ------
def rig_pair(O, S, pf, delay, steps, jitter=0.0, seed=99):
    from paper_2605_16184_b200 import runtime
    opt = runtime.optimizer_defaults(abi.SHAMPOO)
    opt.precondition_frequency = pf
    sched = runtime.scheduler_defaults()
    sched.staleness_S, sched.pf, sched.inject_job_delay_steps = S, pf, delay
    sched.inject_job_delay_jitter_steps = jitter
    sched.step_compute_us, sched.install_cost_us = 1000.0, 5.0
    W = torch.zeros(4, 4, device="cuda")
    G = torch.zeros(4, 4, device="cuda")
    o = O.AsteriaOptimizer([W], [G], opt, sched, seed=seed)
    osched = orc.Scheduler(opt, sched, seed=seed)
    blk = orc.Block(4, 4, abi.SHAMPOO)
    waits_gpu, waits_orc = [], []
    for s in range(steps):
        g = orc.random_matrix(4, 4, 100 + s)
        G.copy_(torch.tensor(g, dtype=torch.float32))
        o.clock_advance(sched.step_compute_us)
        st0 = o.stats().wait_total_us
        o.step(s)
        waits_gpu.append(o.stats().wait_total_us - st0)
        osched.advance(sched.step_compute_us)
        orc.accumulate_factors(blk, g, opt)
        osched.maybe_dispatch(blk, 0, s)
        waits_orc.append(osched.staleness_barrier(blk, 0, s))
        osched.step_end([blk], [0], s)
    o.synchronize()
    return o, osched, waits_gpu, waits_orc


@pytest.mark.parametrize("S,pf,delay,steps,jitter", [
    (5, 10, 0.0, 25, 0.0),    # dispatch cadence          asyncsched_test.cpp:71-76
    (100, 10, 25.0, 30, 0.0),  # coalescing                :78-89
    (0, 10, 2.0, 35, 0.0),    # S=0 every boundary        :91-101
    (3, 10, 2.0, 40, 0.0),    # hidden under budget       :103-115
    (2, 10, 5.0, 20, 0.0),    # barrier at age S+1        :117-129
    (1, 1, 3.0, 40, 0.0),     # consumed age bound        :202-217
    (3, 5, 1.5, 40, 1.5),     # jittered costs (seeded mt19937_64)
])
def test_schedule_matches_oracle(O, S, pf, delay, steps, jitter):
    o, osched, wg, wo = rig_pair(O, S, pf, delay, steps, jitter)
    ev_g = [(e.step, e.kind, e.version, round(e.t_us, 6)) for e in o.events()]
    ev_o = [(e.step, e.kind, e.version, round(e.t_us, 6)) for e in osched.events()]
    assert ev_g == ev_o
    assert np.allclose(wg, wo)
    sg, so = o.stats(), osched.stats()
    assert (sg.dispatched, sg.installed, sg.coalesced, sg.barrier_waits, sg.pending) == \
        (so.dispatched, so.installed, so.coalesced, so.barrier_waits, so.pending)
    fg, fo = o.freshness(0), osched.freshness(0)
    assert (fg.installed_version, fg.dispatch_step_of_pending, fg.last_install_step, fg.installed_snapshot_step) == \
        (fo.installed_version, fo.dispatch_step_of_pending, fo.last_install_step, fo.installed_snapshot_step)


def test_event_mode_bounded_staleness(O):
    from paper_2605_16184_b200 import runtime
    opt = runtime.optimizer_defaults(abi.SOAP)
    opt.precondition_frequency = 2
    sched = runtime.scheduler_defaults()
    sched.staleness_S, sched.pf, sched.install_mode = 1, 2, abi.INSTALL_EVENT
    W = torch.zeros(256, 384, device="cuda")
    G = torch.zeros_like(W)
    o = O.AsteriaOptimizer([W], [G], opt, sched)
    worst = 0
    for s in range(30):
        G.normal_(0, 1e-3)
        o.step(s)
        if o.block_info(0).version > 0:
            worst = max(worst, s - o.freshness(0).installed_snapshot_step)
    o.synchronize()
    st = o.stats()
    assert st.installed >= 10 and st.dispatched == st.installed + st.pending
    assert worst <= (sched.staleness_S + 1) * sched.pf
    assert torch.isfinite(W).all()


def test_event_barrier_does_not_block_and_books_the_device_wait(O):
    """EVENT install mode, S = 0: every step's refresh is installed at the same
    step's barrier (asyncsched.cpp:191-221). The install makes the main stream
    wait on the refresh event instead of blocking the host; the device-side
    wait is measured and booked into wait_total_us at the next host sync."""
    from paper_2605_16184_b200 import runtime
    opt = runtime.optimizer_defaults(abi.SOAP)
    opt.precondition_frequency = 1
    sched = runtime.scheduler_defaults()
    sched.pf, sched.staleness_S, sched.install_mode, sched.refresh_mode = 1, 0, abi.INSTALL_EVENT, abi.REFRESH_F32
    W = (0.1 * torch.randn(512, 512, device="cuda")).contiguous()
    G = torch.randn(512, 512, device="cuda") * 1e-3
    o = O.AsteriaOptimizer([W], [G], opt, sched)
    for step in range(4):
        G.normal_(0.0, 1e-3)
        o.step(step)
    o.synchronize()
    st = o.stats()
    assert st.installed == 4 and st.barrier_waits == 4
    assert st.wait_total_us > 0.0
    assert torch.isfinite(W).all()


def test_non_finite_update_leaves_theta_and_surfaces_at_sync(O):
    """apply_update (precond.cpp:244-251) throws NonFinite without touching
    theta. The fused apply epilogue leaves every non-finite update element's
    theta unchanged, sets the update flag, and the next host sync raises
    NonFiniteError (the gradient-norm flag is separate)."""
    from paper_2605_16184_b200 import runtime
    opt = runtime.optimizer_defaults(abi.SHAMPOO)
    opt.precondition_frequency = 100
    sched = runtime.scheduler_defaults()
    sched.pf, sched.staleness_S = 100, 0
    W = (0.1 * torch.randn(128, 128, device="cuda")).contiguous()
    G = (1e-3 * torch.randn(128, 128, device="cuda")).contiguous()
    o = O.AsteriaOptimizer([W], [G], opt, sched)
    o.step(0)  # refresh dispatched and installed at step 0 (S = 0)
    o.synchronize()
    inv = o.read_block(0, abi.INV_L)
    inv[3, 5] = float("nan")
    import ctypes as C
    runtime.check(runtime.lib.asg_block_write(o._h, 0, abi.INV_L, inv.ctypes.data_as(C.POINTER(C.c_double)), inv.size))
    before = W.clone()
    o.step(1)  # no refresh at step 1: the update uses the poisoned root -> row 3 of U is NaN
    with pytest.raises(abi.NonFiniteError):
        o.synchronize()
    assert torch.equal(W[3], before[3])
    assert torch.isfinite(W).all()
    assert not torch.equal(W[4], before[4])
    o.synchronize()  # flag cleared once reported


def test_synth_gradients_philox_statistics_and_determinism():
    """asg_synth_gradients (the bench's input): every owned block
    slice gets N(0, 1/cols) values, deterministic in (seed, step), fresh per
    step, independent across blocks."""
    import torch
    from paper_2605_16184_b200 import abi, runtime
    from paper_2605_16184_b200.optimizer import AsteriaOptimizer
    opt = runtime.optimizer_defaults(abi.SHAMPOO)
    opt.block_dim_limit = 256
    W = [torch.zeros(512, 768, device="cuda"), torch.zeros(300, device="cuda")]
    G = [torch.zeros_like(w) for w in W]
    o = AsteriaOptimizer(W, G, opt, runtime.scheduler_defaults())
    o.synth_gradients(1234, 7)
    torch.cuda.synchronize()
    a = G[0].clone()
    assert abs(a.mean().item()) < 5e-3 and abs(a.std().item() * 768 ** 0.5 - 1.0) < 1e-2
    b1 = G[1].clone()
    assert abs(b1.std().item() * 300 ** 0.5 - 1.0) < 0.15
    o.synth_gradients(1234, 7)
    torch.cuda.synchronize()
    assert torch.equal(G[0], a)                      # deterministic in (seed, step)
    o.synth_gradients(1234, 8)
    torch.cuda.synchronize()
    assert (G[0] - a).abs().max().item() > 0.1      # fresh every step
    blk = G[0][:256, :256], G[0][:256, 256:512]      # distinct blocks draw distinct streams
    assert not torch.equal(blk[0], blk[1])
    c = torch.corrcoef(torch.stack([blk[0].flatten(), blk[1].flatten()]))[0, 1].item()
    assert abs(c) < 0.02
