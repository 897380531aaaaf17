#!/usr/bin/env python
# SPDX-License-Identifier: Apache-2.0
"""Benchmark of the B200 Asteria optimizer step (SOAP / KL-Shampoo / Shampoo).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3] [--impl ours|reference]

A step = one full optimizer step over the workload's parameter blocks:
fresh synthetic gradients, global-norm clip scale, Kronecker statistics,
bounded-staleness refresh (dispatched every pf steps on a low-priority side
stream), preconditioned update + apply; at N > 1 the blocks are
ownership-sharded and the updated parameters are all-gathered over NCCL.

Gradients are regenerated on the device EVERY step: block b at
step t is N(0, 1/cols) from a Philox generator keyed (1234, t, b), written
by its owner rank inside the timed region (its cost is included and
reported as synth_ms_per_step). The factors therefore change every step and
every refresh does real work (no refresh finds its factor already
diagonal in the previous basis).

Workloads (BASELINE.json configs):
  C1  Shampoo, one 1024x1024 block, EMA b2=0.95, pf=1, S=0 (reference's quadratic_shampoo.json)
  C2  SOAP, GPT-2-small layer set (124M params, block 1024, 171 blocks), pf=10, S=5
  C3  KL-Shampoo, LLaMA-shaped 1B layer set (256 blocks of 2048^2), pf=10, S=5   [default:
      the largest single-GPU config and the north_star target]
  C4  SOAP, the same 256 blocks, ownership-sharded across N GPUs, pf=10, S=5
  C5  the refresh alone: batched eigensolve (--refresh f32) or Newton-Schulz
      inverse roots (--refresh newton) of B_n = 2^31/n^2 factors, n = --n

Prints ONE JSON line on rank 0. `value` is algorithmic TFLOP/s of the whole
job (flop conventions of SURVEY.md 8(d)), `ms_per_step` the step latency.
`--gpus N` without torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU).
"""
import argparse
import json
import math
import os
import socket
import statistics
import subprocess
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


def executed_step_flops(wl):
    """Flops the step's GEMMs execute (the 8(d) products as this library
    forms them). Equal to the convention except KL-Shampoo, whose statistics
    reuse the root P = F^-1/2 (F^-1 = P^2): W = G P_R (2mn^2), L from W W^T
    (m^2 n), V^T = G^T P_L (2m^2 n), R from V^T V (mn^2), update V P_R (2mn^2)
    = 5mn^2 + 3m^2 n instead of 5mn(m+n)."""
    if wl["method"] != "KL-Shampoo":
        return alg_flops(wl)[0]
    return sum(5 * m * n * n + 3 * m * m * n for s in wl["shapes"] for (m, n) in blocks_of(s, wl["limit"]))


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


def traffic_for(workload, precision="3xtf32"):
    """DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per launch of
    the dominant kernel, from the newest committed `ncu --set full` capture
    summary (profiles/r02_traffic.json, else r01; written by profiles/ncu_traffic.py)."""
    key = workload + {"3xtf32_smem": "_smem", "3xf16": "_f16"}.get(precision, "")
    d = None
    for name in ("r02_traffic.json", "r01_traffic.json"):
        p = os.path.join(ROOT, "profiles", name)
        if os.path.exists(p):
            d = json.load(open(p)).get(key)
            if d:
                break
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
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample_shape(wl):
    """The workload's dominant block shape scaled so that one sampled step
    (plus 1/pf of a refresh) is about a second of CPU work: the oracle's
    cyclic Jacobi needs ~20 s per 512^2 factor pair and minutes per 2048^2
    factor."""
    blocks = [b for s in wl["shapes"] for b in blocks_of(s, wl["limit"])]
    m, n = max(set(blocks), key=blocks.count)
    side = 512 if wl["pf"] >= 10 else 256
    f = min(1.0, side / max(m, n))
    return (m, n), (max(8, int(round(m * f))), max(8, int(round(n * f))))


def cpu_baseline(wl, steps, warmup, native=False):
    """The reference path on the host CPU: the fp64 oracle (a restatement of
    the reference's per-block loop, harness.cpp:448-471 with the synchronous
    refresh of reference_opt.cpp:96-99: accumulate_factors, refresh every pf
    steps, precondition, apply_update), built -O3 as the reference's Release
    flags (native=True: the same sources -O3 -march=native, compiled on this
    host), on ONE block of the workload's dominant shape scaled to a bounded
    sample (cpu_sample_shape), with fresh N(0, 1/cols) gradients every step,
    single thread. Each step is one such block step; value is the algorithmic
    flop rate of the timed steps (SURVEY 8(d) conventions for the sampled
    shape), the same metric as the GPU arm; workload_ms_per_step scales the
    measured time to the workload by its block count and shapes (mn(m+n) for
    the step, n^3 for the refresh, refreshes on an nproc-thread pool,
    harness.cpp:312-316)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import orc
    from paper_2605_16184_b200 import abi
    orc.use_build(native)
    meth = {"SOAP": abi.SOAP, "KL-Shampoo": abi.KL_SHAMPOO, "Shampoo": abi.SHAMPOO}[wl["method"]]
    cfg = orc.defaults_for(meth)
    cfg.precondition_frequency = wl["pf"]
    cfg.accumulation = abi.EMA if wl["accumulation"] == "EMA" else abi.SUM
    cfg.lr = wl["lr"]
    (M, N), (m, n) = cpu_sample_shape(wl)
    blk = orc.Block(m, n, meth)
    theta = np.zeros((m, n))
    rng = np.random.default_rng(1234)
    t_step, t_ref, n_ref = 0.0, 0.0, 0
    for k in range(warmup + steps):
        g = rng.standard_normal((m, n)) / math.sqrt(n)
        t0 = time.perf_counter()
        orc.accumulate_factors(blk, g, cfg)
        t1 = time.perf_counter()
        if k % wl["pf"] == 0:
            orc.refresh_inverse(blk, cfg, k)
        t2 = time.perf_counter()
        theta = orc.apply_update(theta, orc.step_update(blk, g, cfg), cfg)
        t3 = time.perf_counter()
        if k >= warmup:
            t_step += (t1 - t0) + (t3 - t2)
            t_ref += t2 - t1
            n_ref += (k % wl["pf"] == 0)
    sample_wl = dict(wl, shapes=[(m, n)], limit=max(m, n))
    st_f, ref_f, _ = alg_flops(sample_wl)
    flops = st_f * steps + ref_f * n_ref
    wall = t_step + t_ref
    cores = os.cpu_count() or 1
    blocks = [b for s in wl["shapes"] for b in blocks_of(s, wl["limit"])]
    step_ps = t_step / steps
    ref_each = t_ref / n_ref if n_ref else 0.0
    w_step = sum(step_ps * (bm * bn * (bm + bn)) / (m * n * (m + n)) for (bm, bn) in blocks)
    w_ref = sum(ref_each * (bm ** 3 + bn ** 3) / (m ** 3 + n ** 3) for (bm, bn) in blocks)
    return {"value": flops / wall / 1e12, "unit": "TFLOP/s", "cores": 1, "kind": "port",
            "ms_per_step": wall * 1e3 / steps, "wall_s": wall,
            "workload_ms_per_step": (w_step + w_ref / wl["pf"] / cores) * 1e3,
            "sample": (f"oracle (fp64 restatement of the reference path, -O3{' -march=native' if native else ''}, "
                       f"{cpu_model()}): {steps} timed steps of one {m}x{n} {wl['method']} block (the workload's "
                       f"dominant {M}x{N} shape scaled to a bounded sample), fresh gradients, {n_ref} synchronous "
                       f"refreshes (cyclic Jacobi) every pf={wl['pf']} steps, single thread; "
                       f"{step_ps*1e3:.1f} ms per block step, {ref_each:.1f} s per refresh")}


def cpu_eigh_baseline(n, batch, native=False, ns=384):
    """The oracle's cyclic Jacobi (densela.hpp:182-264 restated, -O3) on one
    384x384 SPD factor, extrapolated by n^3 and spread over nproc threads (the
    reference's refresh pool, harness.cpp:312-316)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import orc
    orc.use_build(native)
    a = orc.random_spd(ns, 7)
    t0 = time.perf_counter()
    orc.sym_eig(a)
    t1 = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    t_total = t1 * (n / ns) ** 3 * batch / cores
    return {"value": 9.0 * n ** 3 * batch / t_total / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "port",
            "ms_per_step": t_total * 1e3, "sample_wall_s": t1, "extrapolation": t_total / t1,
            "sample": f"oracle cyclic Jacobi (fp64, -O3{' -march=native' if native else ''}, {cpu_model()}) on one "
                      f"{ns}x{ns} SPD factor: {t1*1e3:.0f} ms; extrapolated by n^3 to {batch} factors of n={n} on "
                      f"{cores} threads"}


def run_c5(args, rank, world, local):
    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2605_16184_b200 import abi
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

    newton = args.refresh == "newton"
    # NEWTON iterates: 3xFP16 (auto) or 3xTF32 pairs
    nprec = abi.PREC_3XTF32 if args.precision in ("3xtf32", "3xtf32_smem") else abi.PREC_3XF16

    def solve():
        if not mine:
            return
        if newton:  # KL-Shampoo's L^-1/2 (p = 2) of every factor, relative damping 1e-8
            rt.check(rt.lib.asg_inv_root_batched_f32(C.c_void_p(a.data_ptr()), C.c_void_p(v.data_ptr()), mine, n, 2,
                                                     1e-8, nprec, C.c_void_p(stream.cuda_stream or 1)))
        else:
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
    if newton:  # ||X A X - I|| of the inverse square root
        eye = torch.eye(n, dtype=torch.float64, device=dev)
        eps = 1e-8 * torch.diagonal(ad, dim1=1, dim2=2).sum(-1) / n
        resid = ((vd @ (ad + eps[:, None, None] * eye) @ vd - eye).abs().amax()).item() if k else None
    else:
        resid = ((ad @ vd - vd * w[:k, None, :]).abs().amax() / ad.abs().amax()).item() if k else None
    if rank == 0:
        flops = (10.0 if newton else 9.0) * n ** 3 * total
        peak, _, _, src = measured_peaks()
        line = {"metric": ("batched refresh inverse-root throughput (algorithmic TFLOP/s, 9n^3 + n^3 per factor)"
                           if newton else "batched refresh eigensolve throughput (algorithmic TFLOP/s, 9n^3 per factor)"),
                "value": flops * args.steps / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": (f"f32 ({'3xFP16' if nprec == abi.PREC_3XF16 else '3xTF32'} tcgen05 coupled Newton-Schulz, L^-1/2)"
                          if newton
                          else "f32 (3xTF32 tcgen05 block Jacobi, fp32 pair solves)"),
                "data": "synthetic SPD factors X X^T/2n + 1e-3 I (cold solves)",
                "config": {"workload": WORKLOADS["C5"]["name"], "n": n, "factors": total,
                           "parallelism": f"factor-sharded x{world}" if world > 1 else "single",
                           "l2": "inputs > L2 (8 GiB of factors per step)", "refresh": args.refresh,
                           ("max_abs_XAX_minus_I" if newton else "max_residual_rel"): resid},
                "roofline": {"kernel": ("gemm_tn_kernel EPI_SYM_SPLIT/EPI_NS chain (algorithmic 10n^3 vs tensor peak)"
                                        if newton else "tj_apply_kernel + tj_pair_kernel (algorithmic 9n^3 vs tensor peak)"),
                             "bound": "tensor", "achieved": flops * args.steps / (ms / 1e3) / 1e12 / world,
                             "peak": peak, "unit": "TFLOP/s",
                             "frac": flops * args.steps / (ms / 1e3) / 1e12 / world / peak,
                             "peak_note": f"{src} dense bf16", **traffic_for("C5")},
                "gpu_launches": lc1.value - lc0.value, "clocks": clk.summary(),
                "e2e": None}
        if not args.no_cpu_baseline:
            cb = cpu_eigh_baseline(n, total)  # the reference refresh is an eigendecomposition either way
            line["cpu_baseline"] = {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_distributed(n):
    """`bench.py --gpus N` outside torchrun: one rank per GPU under
    torch.distributed.run (the launch the driver uses)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def pct(xs, q):
    if not xs:
        return None
    xs = sorted(xs)
    k = min(len(xs) - 1, max(0, int(math.ceil(q / 100.0 * len(xs))) - 1))
    return xs[k]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=os.environ.get("ASG_WORKLOAD", "C3"), choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="auto", choices=["auto", "3xtf32", "3xtf32_smem", "3xf16", "tf32"],
                    help="3xtf32: operands stored as (hi, lo) tf32 pairs; 3xtf32_smem: the same products, operands "
                         "stored as plain fp32 and split in shared memory; 3xf16: the step's operands as scaled "
                         "(hi, lo) fp16 pairs (kind::f16, twice the tf32 rate); tf32: one product; auto (default): "
                         "3xf16 for Shampoo / KL-Shampoo, 3xtf32 for SOAP (whose chain 3xf16 does not cover)")
    ap.add_argument("--refresh", default="newton", choices=["newton", "f32", "f64"],
                    help="refresh arithmetic: newton = Newton-Schulz roots for Shampoo/KL (SOAP: f32 eigensolve), "
                         "f32 = fp32-level tensor-core eigensolve, f64 = reference-tight fp64 eigensolve")
    ap.add_argument("--n", type=int, default=2048, help="C5: factor dimension of the sweep point")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--fixed-grads", action="store_true", help="diagnostics: one gradient draw for the whole run")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args.gpus)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.workload == "C5" and args.impl == "ours":
        run_c5(args, rank, world, local)
        return
    if args.precision == "auto":
        args.precision = "3xtf32" if wl["method"] == "SOAP" else "3xf16"
    step_flops, refresh_flops, flops = alg_flops(wl)
    cfg_out = {"workload": wl["name"], "method": wl["method"], "blocks": sum(len(blocks_of(s, wl["limit"])) for s in wl["shapes"]),
               "params": sum(math.prod(s) for s in wl["shapes"]), "block_dim_limit": wl["limit"],
               "pf": wl["pf"], "staleness_S": wl["S"], "precision": args.precision, "refresh": args.refresh,
               "parallelism": f"block-sharded x{world}" if world > 1 else "single",
               "gradients": ("fixed (diagnostics)" if args.fixed_grads else
                             "fresh every step: Philox N(0, 1/cols) keyed (1234, step, block), on the owner"),
               "l2": "inputs > L2 (every step streams all state and gradients from HBM)",
               "alg_tflop_per_step": flops / 1e12,
               "executed_step_tflop": executed_step_flops(wl) / 1e12,
               "flops_note": ("value counts the SURVEY 8(d) convention flops (stats + update + refresh/pf); "
                              "executed_step_tflop is what the step's GEMMs execute (KL-Shampoo forms "
                              "G F^-1 G^T as (G P)(G P)^T with P = F^-1/2, 20% fewer); roofline.achieved "
                              "uses executed flops")}

    if args.impl == "reference":
        if rank != 0:
            return
        if args.workload == "C5":
            total = (1 << 31) // (args.n * args.n)
            cb = cpu_eigh_baseline(args.n, total)
            cfg_out = {"workload": wl["name"], "n": args.n, "factors": total}
            cb["wall_s"] = cb["sample_wall_s"]
            steps_run = 1
        else:
            cb = cpu_baseline(wl, args.steps, args.warmup)
            steps_run = args.steps
        metric = ("batched refresh eigensolve throughput (algorithmic TFLOP/s, 9n^3 per factor)" if args.workload == "C5"
                  else "optimizer step throughput (algorithmic TFLOP/s); step latency in ms_per_step")
        line = {"impl": "reference", "metric": metric,
                "value": cb["value"], "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": steps_run,
                "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": cfg_out,
                "cpu_baseline": {"value": cb["value"], "unit": "TFLOP/s", "cores": cb["cores"], "kind": "port",
                                 "sample": cb["sample"], "wall_s": cb["wall_s"]},
                "note": ("the reference path restated as the fp64 oracle (the reference's own sources are "
                         "unbuildable here: Eigen3 absent, DESIGN.md §4); each step is a bounded sample of the "
                         "workload (see cpu_baseline.sample), value is its algorithmic flop rate and ms_per_step "
                         "its measured time"),
                "e2e": {"value": cb["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        if "workload_ms_per_step" in cb:
            line["workload_ms_per_step_extrapolated"] = cb["workload_ms_per_step"]
        print(json.dumps(line), flush=True)
        return

    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2605_16184_b200 import abi, runtime
    from paper_2605_16184_b200.optimizer import AsteriaOptimizer, stream_arg

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
    sched.refresh_mode = {"f32": abi.REFRESH_F32, "f64": abi.REFRESH_F64, "newton": abi.REFRESH_NEWTON}[args.refresh]
    # The cold first refresh (dispatched at step 0) must be installed before
    # timing: its barrier fires at step S+1, so warm up past it.
    args.warmup = max(args.warmup, wl["S"] + 2)
    prec = {"3xtf32": abi.PREC_3XTF32, "3xtf32_smem": abi.PREC_3XTF32_SMEM, "3xf16": abi.PREC_3XF16,
            "tf32": abi.PREC_TF32}[args.precision]

    gen = torch.Generator(device=dev).manual_seed(1234)
    params, grads = [], []
    for s in wl["shapes"]:
        params.append((torch.randn(*s, device=dev, generator=gen) * 0.02).contiguous())
        grads.append(torch.zeros(*s, device=dev))
    o = AsteriaOptimizer(params, grads, opt, sched, precision=prec, rank=rank, world=world, seed=1234)
    stream = torch.cuda.ExternalStream(o.stream_handle)
    def synth(step):
        """Fresh gradients of this rank's units: N(0, 1/cols), Philox4x32-10 keyed
        (1234, step, block): one fused launch over every owned block (asg_synth_gradients)."""
        o.synth_gradients(1234, step)

    def one_step(step, fresh=True):
        if fresh and not args.fixed_grads:
            synth(step)
        norm = math.sqrt(o.grad_sqnorm())             # D2H of the clip statistic (harness.cpp:435)
        o.step(step, clip_scale=o.clip_scale_from_norm(norm), lr_scale=1.0)
        if world > 1:
            o.allgather()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world > 1:
            t = torch.tensor([x], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t.item()
        return x

    if args.fixed_grads:
        synth(0)
    step = 0
    for _ in range(args.warmup):
        one_step(step)
        step += 1
    barrier()
    # cost of the gradient synthesis alone (reported; it is inside the timed steps)
    cur = torch.cuda.current_stream(dev)
    es0, es1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es0.record(cur)
    for k in range(3):
        synth(10 ** 6 + k)
    es1.record(cur)
    barrier()
    synth_ms = es0.elapsed_time(es1) / 3 if not args.fixed_grads else 0.0

    # ---- timed region: inputs resident in HBM (regenerated on the device each step) ----
    o.profile(True)
    o.kernel_stats(reset=True)
    o.hbm_stats(reset=True)
    st0 = o.stats()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    installs = []
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            evs[k].record(cur)
            i0 = o.stats().installed
            one_step(step)
            installs.append(o.stats().installed - i0)
            step += 1
        # the step (and the last all-gather) end on the caller's stream
        cur.wait_stream(stream)
        evs[-1].record(cur)
        barrier()
    ks = o.kernel_stats(reset=True)
    hb = o.hbm_stats(reset=True)
    o.profile(False)
    st1 = o.stats()
    per_step = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    ms = max_over_ranks(evs[0].elapsed_time(evs[-1]))
    ms_per_step = ms / args.steps
    value = flops * args.steps / (ms / 1e3) / 1e12
    with_inst = [t for t, n in zip(per_step, installs) if n > 0]
    without = [t for t, n in zip(per_step, installs) if n == 0]

    # ---- e2e: each step's gradients from pinned host memory (H2D in the timed
    # region, double-buffered on a copy stream as a data loader would) + D2H of
    # the clip statistic ----
    e2e = None
    if not args.no_e2e:
        stride = o.gather_stride()
        shard = o.shard_elems(rank)
        send = torch.zeros(stride * world, dtype=torch.float32, device=dev)
        ring = []
        for r in range(3):  # three distinct host batches (fresh Philox draws), cycled
            synth(2 * 10 ** 6 + r)
            runtime.check(runtime.lib.asg_pack_grads(o._h, C.c_void_p(send.data_ptr()), stream_arg(cur)))
            h = torch.empty(shard, dtype=torch.float32).pin_memory()
            h.copy_(send[rank * stride: rank * stride + shard])
            ring.append(h)
        del send
        staging = [torch.empty(max(1, shard), dtype=torch.float32, device=dev) for _ in range(2)]
        copy_stream = torch.cuda.Stream(dev)
        ev_copied = [torch.cuda.Event() for _ in range(2)]
        ev_consumed = [torch.cuda.Event() for _ in range(2)]

        def prefetch(k):
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(ev_consumed[k % 2])  # staging free once the step two back took it
                staging[k % 2][:shard].copy_(ring[k % 3], non_blocking=True)
                ev_copied[k % 2].record(copy_stream)

        n_e2e = max(3, args.steps // 2)
        for e in ev_consumed:
            e.record(cur)
        barrier()
        t0 = time.perf_counter()
        prefetch(0)
        for k in range(n_e2e):
            cur.wait_event(ev_copied[k % 2])
            # owner-major segment -> this rank's gradient slices (one kernel)
            runtime.check(runtime.lib.asg_unpack_reduced_grads(o._h, C.c_void_p(staging[k % 2].data_ptr()), 1.0,
                                                               stream_arg(cur)))
            ev_consumed[k % 2].record(cur)
            if k + 1 < n_e2e:
                prefetch(k + 1)
            one_step(step, fresh=False)
            step += 1
        barrier()
        t_e2e = max_over_ranks((time.perf_counter() - t0) * 1e3)
        e2e = {"value": flops * n_e2e / (t_e2e / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": t_e2e / n_e2e,
               "h2d_bytes_per_step": shard * 4, "d2h_bytes_per_step": 12,
               "note": "host-clock over the e2e steps; three distinct pinned host gradient batches cycled"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    peak, peak_sus, hbm, peak_src = measured_peaks()
    ach = ks.gemm_alg_flops / (ks.gemm_ms / 1e3) / 1e12 if ks.gemm_ms > 0 else None
    hbm_kernels = {}
    for name, (nl, nbytes, kms) in hb.items():
        if nl:
            hbm_kernels[name] = {"gbs": nbytes / (kms / 1e3) / 1e9 if kms > 0 else None,
                                 "ms_per_step": kms / args.steps, "bytes_per_launch": nbytes / nl,
                                 "frac_of_hbm_peak": (nbytes / (kms / 1e3) / 1e9 / hbm) if kms > 0 else None}
    line = {
        "metric": "optimizer step throughput (algorithmic TFLOP/s); step latency in ms_per_step",
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": (("f32 (3xFP16 tensor-core products: scaled fp16 (hi, lo) pairs, fp32-faithful; "
                   if prec == abi.PREC_3XF16 else "f32 (3xTF32 tensor-core products; ") +
                  {"f32": "fp32-level refresh: tensor-core block Jacobi)",
                   "newton": "fp32-level refresh: Newton-Schulz roots (SOAP: tensor-core block Jacobi))",
                   "f64": "fp64 refresh)"}[args.refresh] if prec != abi.PREC_TF32 else "tf32"),
        "data": "synthetic (fresh N(0, 1/cols) gradients every step, generated on the device; random-init parameters)",
        "config": cfg_out,
        "step_ms": {"p50": pct(per_step, 50), "p99": pct(per_step, 99),
                    "with_install": {"n": len(with_inst), "p50": pct(with_inst, 50), "p99": pct(with_inst, 99)},
                    "without_install": {"n": len(without), "p50": pct(without, 50), "p99": pct(without, 99)},
                    "per_step": [round(t, 3) for t in per_step], "installs_per_step": installs},
        "synth_ms_per_step": synth_ms,
        "roofline": {"kernel": "tcgen05 TN GEMMs of the step, fused epilogues (refresh GEMMs on the side stream excluded)", "bound": "tensor",
                     "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                     "frac": (ach / peak) if ach else None,
                     "peak_note": f"{peak_src} dense bf16 (MEASURED_PEAKS.json bf16_tflops); tf32 kind = bf16/2, "
                                  f"fp16 kind = bf16; 3xTF32 / 3xFP16 issue 3 MMAs per algorithmic product "
                                  f"(mode peak = bf16/6 / bf16/3)",
                     "frac_of_mode_peak": (ach / (peak / {abi.PREC_TF32: 2, abi.PREC_3XF16: 3}.get(prec, 6)))
                                          if ach else None,
                     "gemm_launches": ks.gemm_launches, "gemm_ms_per_step": ks.gemm_ms / args.steps,
                     **traffic_for(args.workload, args.precision)},
        "hbm_kernels": hbm_kernels,
        "gpu_launches": ks.launches,
        "clocks": clk.summary(),
        "schedule": {"dispatched": st1.dispatched - st0.dispatched, "installed": st1.installed - st0.installed,
                     "barrier_waits": st1.barrier_waits - st0.barrier_waits,
                     "barrier_wait_ms": (st1.wait_total_us - st0.wait_total_us) / 1e3},
        "e2e": e2e,
        "state_bytes": o.state_bytes(),
        "workspace_bytes": o.workspace_bytes(),
    }
    if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
        cb = cpu_baseline(wl, steps=10, warmup=1)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "wall_s",
                                                   "workload_ms_per_step")}
        try:
            cn = cpu_baseline(wl, steps=10, warmup=1, native=True)
            line["cpu_baseline"]["native"] = {k: cn[k] for k in ("value", "wall_s", "sample")}
        except Exception as e:  # -march=native build unavailable on this host
            line["cpu_baseline"]["native"] = {"unavailable": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
