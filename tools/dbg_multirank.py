# Debug: one process, rank 0/1 blocksets of world 2 vs a world-1 blockset, step by step.
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2605_16184_b200 import abi, runtime
from paper_2605_16184_b200.optimizer import AsteriaOptimizer

SHAPES = [(256, 384), (300,), (128, 256), (96, 96)]
opt = runtime.optimizer_defaults(abi.SOAP)
opt.lr, opt.block_dim_limit, opt.precondition_frequency = 1e-2, 128, 2
sched = runtime.scheduler_defaults()
sched.pf, sched.staleness_S = 2, 1
g = torch.Generator().manual_seed(0)
p0 = [(0.1 * torch.randn(*s, generator=g)) for s in SHAPES]
P1 = [p.clone().cuda() for p in p0]
Pr = [[p.clone().cuda() for p in p0] for _ in range(2)]
G = [torch.zeros_like(p) for p in P1]
o1 = AsteriaOptimizer(P1, G, opt, sched, rank=0, world=1)
orr = [AsteriaOptimizer(Pr[r], G, opt, sched, rank=r, world=2) for r in range(2)]
print("owners", [orr[0].block_info(i).owner_rank for i in range(orr[0].num_blocks)])
for step in range(5):
    for gr in G:
        gr.copy_(1e-3 * torch.randn(*gr.shape, generator=g))
    for o in [o1] + orr:
        o.clock_advance(sched.step_compute_us)
        o.step(step)
        o.synchronize()
    torch.cuda.synchronize()
    # compare each rank's OWNED blocks with the single-rank result (before exchange)
    for r in range(2):
        for i in range(orr[r].num_blocks):
            bi = orr[r].block_info(i)
            if bi.owner_rank != r:
                continue
            sp = bi.spec
            a = Pr[r][sp.param_index].reshape(-1, SHAPES[sp.param_index][-1])[sp.row_begin:sp.row_end, sp.col_begin:sp.col_end]
            b = P1[sp.param_index].reshape(-1, SHAPES[sp.param_index][-1])[sp.row_begin:sp.row_end, sp.col_begin:sp.col_end]
            d = (a - b).abs().max().item()
            if d > 0:
                print(f"step {step} rank {r} block {i} param {sp.param_index} rows {sp.row_begin}:{sp.row_end} cols {sp.col_begin}:{sp.col_end} diff {d:.3e}")
    # exchange owned slices (emulated all-gather)
    for i in range(orr[0].num_blocks):
        bi = orr[0].block_info(i)
        src = bi.owner_rank
        sp = bi.spec
        for r in range(2):
            if r != src:
                dst = Pr[r][sp.param_index].view(-1, SHAPES[sp.param_index][-1])
                dst[sp.row_begin:sp.row_end, sp.col_begin:sp.col_end] = Pr[src][sp.param_index].view(-1, SHAPES[sp.param_index][-1])[sp.row_begin:sp.row_end, sp.col_begin:sp.col_end]
    print("step", step, "max diff", max((Pr[0][k] - P1[k]).abs().max().item() for k in range(len(SHAPES))))
