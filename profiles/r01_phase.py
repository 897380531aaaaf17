# SPDX-License-Identifier: Apache-2.0
"""Phase breakdown of the optimizer step on one B200 (profiling tool, not a test).

  python profiles/r01_phase.py eigh   [n ...]     cold batched eigh per dimension
  python profiles/r01_phase.py step   C2|C3 ...   step without refresh / step with a synchronous refresh

Prints one JSON object per measurement (CUDA events on the launching stream).
"""
import ctypes as C
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_16184_b200 import abi, runtime as rt  # noqa: E402


def eigh(ns):
    for n in ns:
        b = max(1, min(64, (1 << 28) // (n * n * 8)))
        x = torch.randn(b, n, 2 * n, dtype=torch.float64, device="cuda")
        a = (x @ x.transpose(1, 2)) / (2 * n) + 1e-3 * torch.eye(n, dtype=torch.float64, device="cuda")
        w = torch.empty(b, n, dtype=torch.float64, device="cuda")
        v = torch.empty(b, n, n, dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream

        def run():
            rt.check(rt.lib.asg_sym_eig_batched(C.c_void_p(a.data_ptr()), C.c_void_p(w.data_ptr()),
                                                C.c_void_p(v.data_ptr()), b, n, C.c_void_p(s)))
        run()
        torch.cuda.synchronize()
        reps = []
        for _ in range(int(os.environ.get("ASG_REPS", 3))):  # min over repetitions
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1))
        ms = min(reps)
        res = (a @ v - v * w[:, None, :]).abs().amax().item() / a.abs().amax().item()
        orth = (v.transpose(1, 2) @ v - torch.eye(n, dtype=torch.float64, device="cuda")).abs().amax().item()
        print(json.dumps(dict(phase="eigh_cold", n=n, batch=b, ms=ms, ms_per_matrix=ms / b,
                              alg_tflops=9 * n ** 3 * b / ms / 1e9, residual=res, orth=orth)), flush=True)


def eigh32(ns):
    """Cold batched eigh through the F32 refresh's tensor-core Jacobi."""
    for n in ns:
        b = max(1, min(512, (1 << 31) // (n * n * 4)))  # 8 GiB fp32 per point at most (C5 sizing)
        b = min(b, int(os.environ.get("ASG_EIGH_BATCH", b)))
        g = torch.Generator(device="cuda").manual_seed(1234 + n)
        x = torch.randn(b, n, 2 * n, dtype=torch.float32, device="cuda", generator=g)
        a = (x @ x.transpose(1, 2)) / (2 * n) + 1e-3 * torch.eye(n, device="cuda")
        del x
        w = torch.empty(b, n, dtype=torch.float64, device="cuda")
        v = torch.empty(b, n, n, dtype=torch.float32, device="cuda")
        s = torch.cuda.current_stream().cuda_stream

        def run():
            rt.check(rt.lib.asg_sym_eig_batched_f32(C.c_void_p(a.data_ptr()), C.c_void_p(w.data_ptr()),
                                                    C.c_void_p(v.data_ptr()), b, n, C.c_void_p(s)))
        run()
        torch.cuda.synchronize()
        reps = []
        for _ in range(int(os.environ.get("ASG_REPS", 3))):  # min over repetitions
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1))
        ms = min(reps)
        k = min(b, 4)
        ad, vd, wd = a[:k].double(), v[:k].double(), w[:k]
        res = (ad @ vd - vd * wd[:, None, :]).abs().amax().item() / ad.abs().amax().item()
        orth = (vd.transpose(1, 2) @ vd - torch.eye(n, dtype=torch.float64, device="cuda")).abs().amax().item()
        print(json.dumps(dict(phase="eigh32_cold", n=n, batch=b, ms=ms, reps=reps, ms_per_matrix=ms / b,
                              alg_tflops=9 * n ** 3 * b / ms / 1e9, residual=res, orth=orth)), flush=True)
        del a, v, w
        torch.cuda.empty_cache()


def step(wls):
    import bench
    for name in wls:
        wl = bench.WORKLOADS[name]
        meth = {"SOAP": abi.SOAP, "KL-Shampoo": abi.KL_SHAMPOO, "Shampoo": abi.SHAMPOO}[wl["method"]]
        gen = torch.Generator(device="cuda").manual_seed(1234)
        params, grads = [], []
        for s in wl["shapes"]:
            params.append((torch.randn(*s, device="cuda", generator=gen) * 0.02).contiguous())
            grads.append((torch.randn(*s, device="cuda", generator=gen) / math.sqrt(s[-1])).contiguous())
        from paper_2605_16184_b200.optimizer import AsteriaOptimizer
        for pf, label, nsteps in ((1 << 40, "step_no_refresh", 5), (1, "step_with_sync_refresh", 3)):
            opt = rt.optimizer_defaults(meth)
            opt.lr, opt.precondition_frequency, opt.block_dim_limit = wl["lr"], pf, wl["limit"]
            opt.accumulation = abi.EMA
            sched = rt.scheduler_defaults()
            sched.pf, sched.staleness_S, sched.install_mode = pf, 0, abi.INSTALL_SIM_CLOCK
            sched.refresh_mode = abi.REFRESH_F32 if os.environ.get("ASG_REFRESH", "f64") == "f32" else abi.REFRESH_F64
            o = AsteriaOptimizer(params, grads, opt, sched, precision=abi.PREC_3XTF32)
            st = torch.cuda.ExternalStream(o.stream_handle)
            o.step(0)  # first step (pf huge: the only dispatch)
            o.synchronize()
            times = []
            for k in range(1, nsteps + 1):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(st)
                t0 = time.perf_counter()
                o.step(k)
                e1.record(st)
                o.synchronize()
                times.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
            print(json.dumps(dict(phase=label, workload=name, refresh=os.environ.get("ASG_REFRESH", "f64"), ms_device=[t[0] for t in times],
                                  ms_wall=[t[1] for t in times])), flush=True)
            del o
            torch.cuda.empty_cache()


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "eigh":
        eigh([int(x) for x in sys.argv[2:]] or [256, 512, 768, 1024, 2048])
    elif what == "eigh32":
        eigh32([int(x) for x in sys.argv[2:]] or [256, 512, 1024, 2048, 4096])
    else:
        step(sys.argv[2:] or ["C2"])
