# SPDX-License-Identifier: Apache-2.0
"""Host logic of ownership sharding on CPU: two gloo ranks
plan independently and must agree; every unit has exactly one owner; LPT
keeps the per-rank cost balanced."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_16184_b200 import abi

GPT2_SMALL = [(768, 2304), (2304,), (768, 768), (768,), (768, 3072), (3072,), (3072, 768), (768,)] * 12 + \
             [(50257, 768), (1024, 768), (768,)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_16184_b200 import runtime as rt
    opt = rt.optimizer_defaults(abi.SOAP)
    opt.block_dim_limit = 1024
    plan = rt.plan_owners(opt, GPT2_SMALL, world)
    plans = [None] * world
    dist.all_gather_object(plans, plan)
    if rank == 0:
        q.put(plans)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_agree_on_a_complete_disjoint_plan(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    plans = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(pl == plans[0] for pl in plans)
    plan = plans[0]
    # 171 preconditioned blocks + 12*4 + 1 one-dimensional AdamW parameters
    assert len(plan) == 171 + 49
    assert set(plan) == set(range(world))


def test_lpt_balances_cost():
    from paper_2605_16184_b200 import runtime as rt
    opt = rt.optimizer_defaults(abi.SOAP)
    opt.block_dim_limit = 2048
    shapes = ([(2048, 2048)] * 4 + [(2048, 8192)] * 2 + [(8192, 2048)]) * 16  # 256 equal blocks
    for world in (1, 2, 4, 8):
        plan = rt.plan_owners(opt, shapes, world)
        counts = [plan.count(r) for r in range(world)]
        assert sum(counts) == 256 and max(counts) == min(counts) == 256 // world
