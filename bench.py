#!/usr/bin/env python
# SPDX-License-Identifier: Apache-2.0
"""Benchmark of the B200 Asteria optimizer step (SOAP / KL-Shampoo / Shampoo).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2] [--impl ours|reference]

A step = one full optimizer step over the workload's parameter blocks:
global-norm clip scale, Kronecker statistics, bounded-staleness refresh
(dispatched every pf steps on a low-priority side stream), preconditioned
update + apply; at N > 1 the blocks are ownership-sharded and the updated
parameters are all-gathered over NCCL. Gradients are synthetic (sigma =
1/sqrt(cols), fixed per run; every step's inputs, > L2, are read from HBM).

Workloads (BASELINE.json configs):
  C1  Shampoo, one 1024x1024 block, EMA b2=0.95, pf=1, S=0 (reference's quadratic_shampoo.json)
  C2  SOAP, GPT-2-small layer set (124M params, block 1024, 171 blocks), pf=10, S=5   [default]
  C3  KL-Shampoo, LLaMA-shaped 1B layer set (256 blocks of 2048^2), pf=10, S=5
  C4  SOAP, the same 256 blocks, ownership-sharded across N GPUs, pf=10, S=5

Prints ONE JSON line on rank 0. `value` is algorithmic TFLOP/s of the whole
job (flop conventions of SURVEY.md 8(d)), `ms_per_step` the step latency.
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def gpt2_small():
    shapes = []
    for _ in range(12):
        shapes += [(768, 2304), (2304,), (768, 768), (768,), (768, 3072), (3072,), (3072, 768), (768,),
                   (768,), (768,), (768,), (768,)]  # + ln_1 / ln_2 weight & bias
    shapes += [(50257, 768), (1024, 768), (768,), (768,)]
    return shapes


def llama_1b():
    shapes = []
    for _ in range(16):
        shapes += [(2048, 2048)] * 4 + [(2048, 8192), (2048, 8192), (8192, 2048)]
    return shapes


WORKLOADS = {
    "C1": dict(name="C1: Shampoo 1024x1024 block (quadratic_shampoo.json hyper-params)", method="Shampoo",
               shapes=[(1024, 1024)], limit=2048, pf=1, S=0, lr=3e-3, accumulation="EMA"),
    "C2": dict(name="C2: SOAP GPT-2-small layer set (124M, block 1024)", method="SOAP", shapes=gpt2_small(),
               limit=1024, pf=10, S=5, lr=1e-3, accumulation="EMA"),
    "C3": dict(name="C3: KL-Shampoo LLaMA-shaped 1B layer set (256 x 2048^2)", method="KL-Shampoo",
               shapes=llama_1b(), limit=2048, pf=10, S=5, lr=1e-3, accumulation="EMA"),
    "C4": dict(name="C4: SOAP LLaMA-shaped 1B layer set (256 x 2048^2), block-sharded", method="SOAP",
               shapes=llama_1b(), limit=2048, pf=10, S=5, lr=1e-3, accumulation="EMA"),
    # C5: the refresh's batched eigensolve alone; a step = one cold solve of
    # B_n = 2^31 / n^2 SPD factors (8 GiB fp32) of dimension --n, split over ranks.
    "C5": dict(name="C5: batched eigh refresh sweep point (B_n = 2^31/n^2 SPD factors)", method="eigh",
               shapes=[], limit=0, pf=1, S=0, lr=0.0, accumulation="EMA"),
}


def blocks_of(shape, limit):
    if len(shape) == 1 or shape[0] == 1 or shape[1] == 1:
        return []
    r, c = shape
    return [(min(r, i + limit) - i, min(c, j + limit) - j) for i in range(0, r, limit) for j in range(0, c, limit)]


def alg_flops(wl):
    """Algorithmic flops per step: stats mn(m+n) (KL: 3mn(m+n));
    update 2mn(m+n) (SOAP: 4mn(m+n)); refresh per pf: eigh 9n^3 per factor,
    + n^3 per reconstructed root / inverse; SOAP re-projection 2m^3+2n^3+4mn(m+n)."""
    step = refresh = 0.0
    meth = wl["method"]
    for s in wl["shapes"]:
        for (m, n) in blocks_of(s, wl["limit"]):
            mn = m * n * (m + n)
            if meth == "SOAP":
                step += mn + 4 * mn
                refresh += 9 * (m ** 3 + n ** 3) + 2 * m ** 3 + 2 * n ** 3 + 4 * mn
            elif meth == "KL-Shampoo":
                step += 3 * mn + 2 * mn
                refresh += 9 * (m ** 3 + n ** 3) + 2 * (m ** 3 + n ** 3)
            else:
                step += mn + 2 * mn
                refresh += 9 * (m ** 3 + n ** 3) + (m ** 3 + n ** 3)
    return step, refresh, step + refresh / wl["pf"]


# ---------------------------------------------------------------------------
# clocks (sampled during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


def traffic_for(workload):
    """DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per launch of
    the dominant kernel, from the committed `ncu --set full` capture summary
    (profiles/r01_traffic.json, written by profiles/ncu_traffic.py)."""
    p = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if not os.path.exists(p):
        return {"traffic": None}
    d = json.load(open(p)).get(workload)
    if not d:
        return {"traffic": None}
    return {"traffic": d["dram_bytes_per_launch"], "traffic_kernel": d["kernel"],
            "traffic_alg_bytes": d.get("alg_bytes_per_launch"), "traffic_source": d["source"]}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU baseline (oracle port; test infrastructure, used only as the timed CPU leg)
# ---------------------------------------------------------------------------
def cpu_baseline(wl, budget_s=20.0):
    """Times the fp64 oracle (a restatement of the reference's hot path, built
    -O3 as the reference's Release flags) on a bounded sample and extrapolates
    to the workload: per-block step work scales as mn(m+n), refresh as n^3
    (Jacobi); the step runs single-threaded per rank (harness.cpp:448), the
    refresh on a pool of nproc threads (harness.cpp:312-316)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import orc
    from paper_2605_16184_b200 import abi
    meth = {"SOAP": abi.SOAP, "KL-Shampoo": abi.KL_SHAMPOO, "Shampoo": abi.SHAMPOO}[wl["method"]]
    cfg = orc.defaults_for(meth)
    cfg.precondition_frequency = wl["pf"]
    ns = 384  # sample block side
    blk = orc.Block(ns, ns, meth)
    theta = np.zeros((ns, ns))
    g = orc.random_matrix(ns, ns, 1) / math.sqrt(ns)
    # warm factors, then time the per-step path
    orc.accumulate_factors(blk, g, cfg)
    orc.refresh_inverse(blk, cfg, 0)
    t0 = time.perf_counter()
    nstep = 0
    while time.perf_counter() - t0 < budget_s / 2 or nstep < 1:
        orc.accumulate_factors(blk, g, cfg)
        upd = orc.step_update(blk, g, cfg)
        theta = orc.apply_update(theta, upd, cfg)
        nstep += 1
    t_step = (time.perf_counter() - t0) / nstep
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    nref = 0
    while time.perf_counter() - t0 < budget_s / 2 or nref < 1:
        orc.refresh_inverse(blk, cfg, 1)
        nref += 1
    t_ref = (time.perf_counter() - t0) / nref
    step_units = ns * ns * 2 * ns
    ref_units = 2 * ns ** 3
    tot_step = tot_ref = 0.0
    for s in wl["shapes"]:
        for (m, n) in blocks_of(s, wl["limit"]):
            tot_step += t_step * (m * n * (m + n)) / step_units
            tot_ref += t_ref * (m ** 3 + n ** 3) / ref_units
    t_per_step = tot_step + tot_ref / wl["pf"] / cores
    _, _, flops = alg_flops(wl)
    return {"value": flops / t_per_step / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "port",
            "ms_per_step": t_per_step * 1e3,
            "sample": (f"oracle (fp64 restatement, -O3) on one {ns}x{ns} {wl['method']} block: {nstep} steps "
                       f"single-thread ({t_step*1e3:.1f} ms/step) + {nref} refreshes ({t_ref*1e3:.0f} ms, Jacobi); "
                       f"extrapolated to the workload by mn(m+n) (step) and n^3 (refresh on {cores} threads, "
                       f"amortized over pf={wl['pf']})")}


# ---------------------------------------------------------------------------
# C5: batched eigensolve sweep point
# ---------------------------------------------------------------------------
def cpu_eigh_baseline(n, batch, budget_s=20.0):
    """The oracle's cyclic Jacobi (densela.hpp:182-264 restated, -O3) on one
    384x384 SPD factor, extrapolated by n^3 and spread over nproc threads (the
    reference's refresh pool, harness.cpp:312-316)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import orc
    ns = 384
    a = orc.random_spd(ns, 7)
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < budget_s or k < 1:
        orc.sym_eig(a)
        k += 1
    t1 = (time.perf_counter() - t0) / k
    cores = os.cpu_count() or 1
    t_total = t1 * (n / ns) ** 3 * batch / cores
    return {"value": 9.0 * n ** 3 * batch / t_total / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "port",
            "ms_per_step": t_total * 1e3,
            "sample": f"oracle cyclic Jacobi (fp64, -O3) on one {ns}x{ns} SPD factor: {k} solves, {t1*1e3:.0f} ms "
                      f"each; extrapolated by n^3 to {batch} factors of n={n} on {cores} threads"}


def run_c5(args, rank, world, local):
    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2605_16184_b200 import runtime as rt
    n = args.n
    total = (1 << 31) // (n * n)
    per = (total + world - 1) // world
    mine = max(0, min(per, total - rank * per))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    a = torch.empty(mine, n, n, dtype=torch.float32, device=dev)
    for i in range(0, mine, 64):  # SPD factors A = X X^T / 2n + 1e-3 I (test_util.hpp:20-26 shape)
        x = torch.randn(min(64, mine - i), n, 2 * n, device=dev, generator=gen)
        a[i:i + 64] = torch.baddbmm(1e-3 * torch.eye(n, device=dev).expand(x.shape[0], n, n), x, x.transpose(1, 2),
                                    alpha=1.0 / (2 * n))
        del x
    w = torch.empty(mine, n, dtype=torch.float64, device=dev)
    v = torch.empty(mine, n, n, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def solve():
        if mine:
            rt.check(rt.lib.asg_sym_eig_batched_f32(C.c_void_p(a.data_ptr()), C.c_void_p(w.data_ptr()),
                                                    C.c_void_p(v.data_ptr()), mine, n, C.c_void_p(stream.cuda_stream or 1)))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        solve()
    barrier()
    lc0, lc1 = C.c_uint64(), C.c_uint64()
    rt.check(rt.lib.asg_launch_count(C.byref(lc0)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            solve()
        e1.record(stream)
        barrier()
    rt.check(rt.lib.asg_launch_count(C.byref(lc1)))
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    k = min(mine, 2)
    ad, vd = a[:k].double(), v[:k].double()
    resid = ((ad @ vd - vd * w[:k, None, :]).abs().amax() / ad.abs().amax()).item() if k else None
    if rank == 0:
        flops = 9.0 * n ** 3 * total
        peak, _, _, src = measured_peaks()
        line = {"metric": "batched refresh eigensolve throughput (algorithmic TFLOP/s, 9n^3 per factor)",
                "value": flops * args.steps / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 (3xTF32 tcgen05 block Jacobi, fp32 pair solves)",
                "data": "synthetic SPD factors X X^T/2n + 1e-3 I (cold solves)",
                "config": {"workload": WORKLOADS["C5"]["name"], "n": n, "factors": total,
                           "parallelism": f"factor-sharded x{world}" if world > 1 else "single",
                           "l2": "inputs > L2 (8 GiB of factors per step)", "max_residual_rel": resid},
                "roofline": {"kernel": "tj_apply_kernel + tj_pair_kernel (algorithmic 9n^3 vs tensor peak)",
                             "bound": "tensor", "achieved": flops * args.steps / (ms / 1e3) / 1e12 / world,
                             "peak": peak, "unit": "TFLOP/s",
                             "frac": flops * args.steps / (ms / 1e3) / 1e12 / world / peak,
                             "peak_note": f"{src} dense bf16", **traffic_for("C5")},
                "gpu_launches": lc1.value - lc0.value, "clocks": clk.summary(),
                "e2e": None}
        if not args.no_cpu_baseline:
            cb = cpu_eigh_baseline(n, total)
            line["cpu_baseline"] = {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=os.environ.get("ASG_WORKLOAD", "C2"), choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "tf32"])
    ap.add_argument("--refresh", default="f32", choices=["f32", "f64"],
                    help="refresh arithmetic: f32 = fp32-level tensor-core refresh (default), "
                         "f64 = reference-tight fp64 eigensolve")
    ap.add_argument("--n", type=int, default=2048, help="C5: factor dimension of the sweep point")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload == "C5" and args.impl == "ours":
        run_c5(args, rank, world, local)
        return
    step_flops, refresh_flops, flops = alg_flops(wl)
    cfg_out = {"workload": wl["name"], "method": wl["method"], "blocks": sum(len(blocks_of(s, wl["limit"])) for s in wl["shapes"]),
               "params": sum(math.prod(s) for s in wl["shapes"]), "block_dim_limit": wl["limit"],
               "pf": wl["pf"], "staleness_S": wl["S"], "precision": args.precision, "refresh": args.refresh,
               "parallelism": f"block-sharded x{args.gpus}" if args.gpus > 1 else "single",
               "l2": "inputs > L2 (every step streams all state and gradients from HBM)",
               "alg_tflop_per_step": flops / 1e12}

    if args.impl == "reference":
        if rank != 0:
            return
        if args.workload == "C5":
            total = (1 << 31) // (args.n * args.n)
            cb = cpu_eigh_baseline(args.n, total, budget_s=max(10.0, 3.0 * args.steps))
            cfg_out = {"workload": wl["name"], "n": args.n, "factors": total}
        else:
            cb = cpu_baseline(wl, budget_s=max(10.0, 3.0 * args.steps))
        metric = ("batched refresh eigensolve throughput (algorithmic TFLOP/s, 9n^3 per factor)" if args.workload == "C5"
                  else "optimizer step throughput (algorithmic TFLOP/s); step latency in ms_per_step")
        line = {"impl": "reference", "metric": metric,
                "value": cb["value"], "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": cfg_out,
                "cpu_baseline": {"value": cb["value"], "unit": "TFLOP/s", "cores": cb["cores"], "kind": "port",
                                 "sample": cb["sample"]},
                "e2e": {"value": cb["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2605_16184_b200 import abi, runtime
    from paper_2605_16184_b200.optimizer import AsteriaOptimizer

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    meth = {"SOAP": abi.SOAP, "KL-Shampoo": abi.KL_SHAMPOO, "Shampoo": abi.SHAMPOO}[wl["method"]]
    opt = runtime.optimizer_defaults(meth)
    opt.lr = wl["lr"]
    opt.precondition_frequency = wl["pf"]
    opt.block_dim_limit = wl["limit"]
    opt.accumulation = abi.EMA if wl["accumulation"] == "EMA" else abi.SUM
    sched = runtime.scheduler_defaults()
    sched.pf, sched.staleness_S = wl["pf"], wl["S"]
    sched.install_mode = abi.INSTALL_EVENT if wl["S"] > 0 else abi.INSTALL_SIM_CLOCK
    sched.refresh_mode = abi.REFRESH_F32 if args.refresh == "f32" else abi.REFRESH_F64
    # The cold first refresh (dispatched at step 0, no previous basis) must be
    # installed before timing: its barrier fires at step S+1, so warm up past it.
    args.warmup = max(args.warmup, wl["S"] + 2)
    prec = abi.PREC_3XTF32 if args.precision == "3xtf32" else abi.PREC_TF32

    gen = torch.Generator(device=dev).manual_seed(1234)
    params, grads = [], []
    for s in wl["shapes"]:
        cols = s[-1]
        params.append((torch.randn(*s, device=dev, generator=gen) * 0.02).contiguous())
        grads.append((torch.randn(*s, device=dev, generator=gen) / math.sqrt(cols)).contiguous())
    o = AsteriaOptimizer(params, grads, opt, sched, precision=prec, rank=rank, world=world, seed=1234)
    stream = torch.cuda.ExternalStream(o.stream_handle)

    def one_step(step):
        norm = math.sqrt(o.grad_sqnorm())             # D2H of the clip statistic (harness.cpp:435)
        o.step(step, clip_scale=o.clip_scale_from_norm(norm), lr_scale=1.0)
        if world > 1:
            o.allgather()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    step = 0
    for _ in range(args.warmup):
        one_step(step)
        step += 1
    barrier()

    # ---- timed region: inputs resident in HBM ----
    o.profile(True)
    o.kernel_stats(reset=True)
    st0 = o.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        t_wall0 = time.perf_counter()
        for _ in range(args.steps):
            one_step(step)
            step += 1
        # the last all-gather runs on the caller's stream: end the region after it
        cur = torch.cuda.current_stream(dev)
        cur.wait_stream(stream)
        e1.record(cur)
        stream.wait_stream(cur)
        barrier()
        t_wall = time.perf_counter() - t_wall0
    ks = o.kernel_stats(reset=True)
    o.profile(False)
    st1 = o.stats()
    ms = e0.elapsed_time(e1)
    ms = max(ms, t_wall * 1e3 * 0.0)  # device-timed
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    ms_per_step = ms / args.steps
    value = flops * args.steps / (ms / 1e3) / 1e12

    # ---- e2e: pinned H2D of each step's gradients + D2H of the clip statistic ----
    e2e = None
    if not args.no_e2e:
        # Each step's gradients arrive from pinned host memory. The H2D of step
        # k+1 streams into a staging buffer on a copy stream while step k
        # computes (double buffering, as a data loader would); step k+1 then
        # moves them into the bound gradient tensors with a device copy.
        # One flat pinned host batch (as a data loader would hand over) and one
        # flat device staging buffer: a single large DMA per step instead of one
        # copy per parameter tensor.
        total = sum(g.numel() for g in grads)
        host_flat = torch.empty(total, dtype=torch.float32).pin_memory()
        staging_flat = torch.empty(total, dtype=torch.float32, device=dev)
        staging, off = [], 0
        for g in grads:
            host_flat[off:off + g.numel()].copy_(g.reshape(-1).cpu())
            staging.append(staging_flat[off:off + g.numel()].view_as(g))
            off += g.numel()
        h2d = total * 4
        copy_stream = torch.cuda.Stream(dev)
        ev_copied, ev_consumed = torch.cuda.Event(), torch.cuda.Event()
        cur = torch.cuda.current_stream(dev)

        def prefetch():
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(ev_consumed)  # staging free once the previous step took it
                staging_flat.copy_(host_flat, non_blocking=True)
                ev_copied.record(copy_stream)

        n_e2e = max(3, args.steps // 2)
        ev_consumed.record(cur)
        barrier()
        t0 = time.perf_counter()
        prefetch()
        for k in range(n_e2e):
            cur.wait_event(ev_copied)
            for g, st_ in zip(grads, staging):
                g.copy_(st_, non_blocking=True)
            ev_consumed.record(cur)
            if k + 1 < n_e2e:
                prefetch()
            one_step(step)
            step += 1
        barrier()
        t_e2e = (time.perf_counter() - t0) * 1e3
        if world > 1:
            t = torch.tensor([t_e2e], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = t.item()
        e2e = {"value": flops * n_e2e / (t_e2e / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": t_e2e / n_e2e,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 12}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    peak, peak_sus, hbm, peak_src = measured_peaks()
    ach = ks.gemm_alg_flops / (ks.gemm_ms / 1e3) / 1e12 if ks.gemm_ms > 0 else None
    line = {
        "metric": "optimizer step throughput (algorithmic TFLOP/s); step latency in ms_per_step",
        "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": ("f32 (3xTF32 tensor-core products; " +
                  ("fp32-level refresh: tensor-core block Jacobi)" if args.refresh == "f32" else "fp64 refresh)")
                  if prec == abi.PREC_3XTF32 else "tf32"),
        "data": "synthetic (N(0, 1/cols) gradients, fixed per run; random-init parameters)",
        "config": cfg_out,
        "roofline": {"kernel": "tcgen05 TN GEMMs of the step, fused epilogues (refresh GEMMs on the side stream excluded)", "bound": "tensor",
                     "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                     "frac": (ach / peak) if ach else None,
                     "peak_note": f"{peak_src} dense bf16 (MEASURED_PEAKS.json bf16_tflops); tf32 kind = bf16/2, "
                                  f"3xTF32 issues 3 tf32 MMAs per algorithmic product",
                     "frac_of_mode_peak": (ach / (peak / 2 / (3 if prec == abi.PREC_3XTF32 else 1))) if ach else None,
                     "gemm_launches": ks.gemm_launches, "gemm_ms_per_step": ks.gemm_ms / args.steps,
                     **traffic_for(args.workload)},
        "gpu_launches": ks.launches,
        "clocks": clk.summary(),
        "schedule": {"dispatched": st1.dispatched - st0.dispatched, "installed": st1.installed - st0.installed,
                     "barrier_waits": st1.barrier_waits - st0.barrier_waits},
        "e2e": e2e,
        "state_bytes": o.state_bytes(),
    }
    if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
        cb = cpu_baseline(wl)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
