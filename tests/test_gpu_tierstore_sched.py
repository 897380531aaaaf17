# SPDX-License-Identifier: Apache-2.0
"""F3 on the optimizer path: a blockset with an attached tier store mirrors
ShadowScheduler's store traffic (asyncsched.cpp:164-184 install write-back and
Hot prefetch, :223-246 ForwardPost drain, :247-267 BackwardPre re-prefetch of
Cold inverse state), with the Hot tier in HBM."""
import numpy as np
import pytest

from paper_2605_16184_b200 import abi
from paper_2605_16184_b200 import trace as T

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _bid(o, i):  # the runtime's unit id: BlockSpec::id with the parameter named w<index>
    return T.block_id(o.block_info(i).spec, param_names=["w0"])


@pytest.mark.parametrize("method,refresh", [(abi.SHAMPOO, abi.REFRESH_NEWTON), (abi.SOAP, abi.REFRESH_F32),
                                            (abi.KL_SHAMPOO, abi.REFRESH_NEWTON)])
def test_installs_write_back_to_the_store_and_drain_to_hbm(tmp_path, method, refresh):
    from paper_2605_16184_b200 import runtime
    from paper_2605_16184_b200.optimizer import AsteriaOptimizer
    from paper_2605_16184_b200.tierstore import TierStore
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    opt = runtime.optimizer_defaults(method)
    opt.block_dim_limit, opt.precondition_frequency = 128, 2
    sched = runtime.scheduler_defaults()
    sched.pf, sched.staleness_S, sched.refresh_mode = 2, 1, refresh
    sched.drain_budget = 8
    g = torch.Generator(device="cuda").manual_seed(3)
    params = [torch.randn(256, 128, device="cuda", generator=g) * 0.1]
    grads = [torch.zeros_like(params[0])]
    o = AsteriaOptimizer(params, grads, opt, sched)
    store = TierStore(str(tmp_path / "opt.cold"), hot_device=0)
    o.attach_store(store)
    roles = (abi.BASIS_L, abi.BASIS_R) if method == abi.SOAP else (abi.INV_L, abi.INV_R)
    steps = 9
    for s in range(steps):
        o.on_hook(abi.HOOK_FORWARD_POST, s)
        o.on_hook(abi.HOOK_BACKWARD_PRE, s)
        grads[0].normal_(generator=g).mul_(1e-3)
        o.step(s)  # accumulate, dispatch, barrier, update, StepEnd
    o.synchronize()
    kinds = [e.kind for e in o.events()]
    assert abi.EV_PREFETCH in kinds and abi.EV_DRAIN in kinds
    # the store holds each block's installed inverse state, byte-exact: (hi | lo) padded fp32 slabs
    nb = o.num_blocks
    for i in range(nb):
        bid = _bid(o, i)
        for side, role in enumerate(roles):
            assert store.contains((bid, role))
            payload, tier = store.get((bid, role))
            assert tier in (abi.TIER_HOT, abi.TIER_HOST)
            ref = o.read_block(i, role)  # fp64 (hi + lo) of the installed state
            d = ref.shape[0]
            D = int(np.sqrt(len(payload) // 8))  # hi and lo slabs of D x D fp32
            a = np.frombuffer(payload, dtype=np.float32).reshape(2, D, D).astype(np.float64)
            np.testing.assert_array_equal((a[0] + a[1])[:d, :d], ref)
    # a Cold entry: BackwardPre re-prefetches it to Host, ForwardPost drains it
    # (first let the install-time Hot prefetches land: a new prefetch of a key
    # with a transfer in flight coalesces onto it, tierstore.cpp:298-302)
    bid = _bid(o, 0)
    for k in range(1, 6):
        o.on_hook(abi.HOOK_FORWARD_POST, steps + k)
    v = store.inspect((bid, roles[0]))
    assert v.tier == abi.TIER_HOT and not v.staged_pending and not v.staged_ready
    store.demote((bid, roles[0]), abi.TIER_COLD)
    n_ev = len(o.events())
    o.on_hook(abi.HOOK_BACKWARD_PRE, steps + 6)
    new = [e.kind for e in o.events()[n_ev:]]
    assert new.count(abi.EV_PREFETCH) == 1
    o.on_hook(abi.HOOK_FORWARD_POST, steps + 7)
    assert store.inspect((bid, roles[0])).tier == abi.TIER_HOST
    store.audit()
    o.attach_store(None)
    store.close()
