# SPDX-License-Identifier: Apache-2.0
"""Block-sharded step + owner-major all-gather on one GPU:
two ranks (gloo, both on cuda:0) each update only their owned blocks and
exchange them; the result must equal a single-rank run bit for bit, because
every block is computed by the same kernels on the same inputs."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SHAPES = [(256, 384), (300,), (128, 256), (96, 96)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank, world, steps):
    from paper_2605_16184_b200 import abi, runtime
    from paper_2605_16184_b200.optimizer import AsteriaOptimizer
    opt = runtime.optimizer_defaults(abi.SOAP)
    opt.lr, opt.block_dim_limit, opt.precondition_frequency = 1e-2, 128, 2
    sched = runtime.scheduler_defaults()
    sched.pf, sched.staleness_S = 2, 1
    g = torch.Generator().manual_seed(0)
    params = [(0.1 * torch.randn(*s, generator=g)).cuda() for s in SHAPES]
    grads = [torch.zeros_like(p) for p in params]
    o = AsteriaOptimizer(params, grads, opt, sched, rank=rank, world=world)
    for step in range(steps):
        for gr in grads:
            gr.copy_(1e-3 * torch.randn(*gr.shape, generator=g))
        o.clock_advance(sched.step_compute_us)
        o.step(step)
        o.allgather()
    o.synchronize()
    return [p.cpu().numpy() for p in params], [o.block_info(i).owner_rank for i in range(o.num_blocks)]


def _worker(rank, world, port, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out, owners = _run(rank, world, steps)
    q.put((rank, out, owners))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_match_single_rank():
    import torch.multiprocessing as mp
    steps = 5
    ref, _ = _run(0, 1, steps)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(2):
        rank, out, owners = q.get(timeout=600)
        results[rank] = (out, owners)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    owners = results[0][1]
    assert set(owners) == {0, 1}  # both ranks own work
    for rank in (0, 1):
        for a, b in zip(results[rank][0], ref):
            assert np.array_equal(a, b), np.abs(a - b).max()
