# SPDX-License-Identifier: Apache-2.0
"""Drives a few optimizer steps of a bench workload so ncu can list every
kernel launch (profiling tool, not a test; run under
`ncu --metrics gpu__time_duration.sum --clock-control none --csv`).

  python profiles/r01_steplaunch.py C2|C3 [pf] [steps]

With pf > steps only step 0 dispatches a refresh (cold); with pf=1 every
step runs a synchronous (S=0) refresh, warm-started after the first.
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_16184_b200 import abi, runtime as rt  # noqa: E402
from paper_2605_16184_b200.optimizer import AsteriaOptimizer  # noqa: E402


def main():
    name = sys.argv[1]
    pf = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 40
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    wl = bench.WORKLOADS[name]
    meth = {"SOAP": abi.SOAP, "KL-Shampoo": abi.KL_SHAMPOO, "Shampoo": abi.SHAMPOO}[wl["method"]]
    gen = torch.Generator(device="cuda").manual_seed(1234)
    params, grads = [], []
    for s in wl["shapes"]:
        params.append((torch.randn(*s, device="cuda", generator=gen) * 0.02).contiguous())
        grads.append((torch.randn(*s, device="cuda", generator=gen) / math.sqrt(s[-1])).contiguous())
    opt = rt.optimizer_defaults(meth)
    opt.lr, opt.precondition_frequency, opt.block_dim_limit = wl["lr"], pf, wl["limit"]
    opt.accumulation = abi.EMA
    sched = rt.scheduler_defaults()
    sched.pf, sched.staleness_S, sched.install_mode = pf, 0, abi.INSTALL_SIM_CLOCK
    sched.refresh_mode = abi.REFRESH_F64 if os.environ.get("ASG_REFRESH", "f32") == "f64" else abi.REFRESH_F32
    o = AsteriaOptimizer(params, grads, opt, sched, precision=abi.PREC_3XTF32)
    for k in range(steps):
        torch.cuda.nvtx.range_push(f"step{k}")
        o.step(k)
        o.synchronize()
        torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    main()
