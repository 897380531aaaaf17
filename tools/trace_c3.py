"""Kernel timeline of the C3 step around a refresh dispatch (torch.profiler /
CUPTI sees every kernel this library launches, on every stream)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_16184_b200 import abi, runtime
from paper_2605_16184_b200.optimizer import AsteriaOptimizer
wl = bench.WORKLOADS["C3"]
dev = torch.device("cuda", 0)
opt = runtime.optimizer_defaults(abi.KL_SHAMPOO)
opt.lr, opt.precondition_frequency, opt.block_dim_limit = wl["lr"], wl["pf"], wl["limit"]
sched = runtime.scheduler_defaults()
sched.pf, sched.staleness_S, sched.install_mode, sched.refresh_mode = 10, 5, abi.INSTALL_EVENT, abi.REFRESH_NEWTON
params = [torch.randn(*s, device=dev) * 0.02 for s in wl["shapes"]]
grads = [torch.randn(*s, device=dev) / math.sqrt(s[-1]) for s in wl["shapes"]]
o = AsteriaOptimizer(params, grads, opt, sched)
for step in range(9):
    for g in grads: g.normal_(0, 0.02)
    o.step(step, clip_scale=o.clip_scale_from_norm(math.sqrt(o.grad_sqnorm())))
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for step in range(9, 13):
        for g in grads: g.normal_(0, 0.02)
        o.step(step, clip_scale=o.clip_scale_from_norm(math.sqrt(o.grad_sqnorm())))
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/c3_trace.json")
ev = json.load(open("gpurun_out/c3_trace.json"))["traceEvents"]
k = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in k)
streams = {}
for e in k:
    streams.setdefault(e["args"].get("stream"), []).append(e)
for sid, es in streams.items():
    es.sort(key=lambda e: e["ts"])
    busy = sum(e["dur"] for e in es)
    print(f"stream {sid}: {len(es)} ops, busy {busy/1e3:.1f} ms, span {(es[0]['ts']-t0)/1e3:.1f}-{(es[-1]['ts']+es[-1]['dur']-t0)/1e3:.1f} ms")
# main-stream gemm gaps
for sid, es in streams.items():
    names = {}
    for e in es:
        n = e["name"].split("<")[0][:40]
        names[n] = names.get(n, 0) + e["dur"]
    print(sid, sorted(names.items(), key=lambda x: -x[1])[:6])
# timeline of big gaps in each stream
for sid, es in streams.items():
    gaps = [(es[i]["ts"] - (es[i-1]["ts"] + es[i-1]["dur"]), i) for i in range(1, len(es))]
    gaps.sort(reverse=True)
    print(sid, "largest gaps (ms, before op):", [(round(g/1e3, 1), es[i]["name"][:30], round((es[i]['ts']-t0)/1e3,1)) for g, i in gaps[:5]])
