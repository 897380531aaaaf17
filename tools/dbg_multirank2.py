# Debug: the gloo two-process version of tests/test_gpu_multirank.py, per-step comparison.
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_multirank as T  # noqa: E402


def run_steps(rank, world, steps, q=None):
    from paper_2605_16184_b200 import abi, runtime
    from paper_2605_16184_b200.optimizer import AsteriaOptimizer
    opt = runtime.optimizer_defaults(abi.SOAP)
    opt.lr, opt.block_dim_limit, opt.precondition_frequency = 1e-2, 128, 2
    sched = runtime.scheduler_defaults()
    sched.pf, sched.staleness_S = 2, 1
    g = torch.Generator().manual_seed(0)
    params = [(0.1 * torch.randn(*s, generator=g)).cuda() for s in T.SHAPES]
    grads = [torch.zeros_like(p) for p in params]
    o = AsteriaOptimizer(params, grads, opt, sched, rank=rank, world=world)
    hist = []
    for step in range(steps):
        for gr in grads:
            gr.copy_(1e-3 * torch.randn(*gr.shape, generator=g))
        o.clock_advance(sched.step_compute_us)
        o.step(step)
        if os.environ.get("SYNC_AFTER_STEP"):
            torch.cuda.synchronize()
        pre = [p.cpu().numpy().copy() for p in params]
        o.allgather()
        o.synchronize()
        hist.append((pre, [p.cpu().numpy().copy() for p in params]))
    owners = [o.block_info(i).owner_rank for i in range(o.num_blocks)]
    specs = [(o.block_info(i).spec.param_index, o.block_info(i).spec.row_begin, o.block_info(i).spec.row_end,
              o.block_info(i).spec.col_begin, o.block_info(i).spec.col_end) for i in range(o.num_blocks)]
    return hist, owners, specs


def worker(rank, world, port, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hist, owners, specs = run_steps(rank, world, steps)
    q.put((rank, hist, owners, specs))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    steps = 5
    ref, _, specs = run_steps(0, 1, steps)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = T._free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, hist, owners, specs2 = q.get(timeout=600)
        res[rank] = (hist, owners)
    for p in procs:
        p.join(timeout=120)
    owners = res[0][1]
    print("owners", owners)
    for step in range(steps):
        d = max(np.abs(a - b).max() for a, b in zip(ref[step][0], ref[step][1]))
        if d > 0:
            print(f"step {step} ref pre/post differ {d:.3e}")
        for r in range(2):
            pre, post = res[r][0][step]
            rpre, rpost = ref[step]
            for bi, (pi, r0, r1, c0, c1) in enumerate(specs):
                shp = T.SHAPES[pi]
                a = pre[pi].reshape(-1, shp[-1])[r0:r1, c0:c1]
                b = rpre[pi].reshape(-1, shp[-1])[r0:r1, c0:c1]
                a2 = post[pi].reshape(-1, shp[-1])[r0:r1, c0:c1]
                b2 = rpost[pi].reshape(-1, shp[-1])[r0:r1, c0:c1]
                d, d2 = np.abs(a - b).max(), np.abs(a2 - b2).max()
                if d > 0 or d2 > 0:
                    print(f"step {step} rank {r} block {bi} owner {owners[bi]} pre-gather diff {d:.3e} post {d2:.3e}")
