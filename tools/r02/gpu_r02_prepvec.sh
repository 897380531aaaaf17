# Vectorised 3xFP16 gradient prep: storage-mode trajectories + f16 GEMM parity, C3 bench, launch list.
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py -m gpu -q --tb=short -k "operand_storage_modes or gemm or synth" 2>&1 | tail -4
timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/r02_pv_C3.jsonl 2> gpurun_out/r02_pv_C3.err
python - gpurun_out/r02_pv_C3.jsonl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), d["step_ms"]["p50"], r["gemm_ms_per_step"], d["clocks"], d["e2e"]["ms_per_step"], d["schedule"]["barrier_waits"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
tail -2 gpurun_out/r02_pv_C3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_pv_launches.csv python bench.py --workload C3 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(open("gpurun_out/r02_pv_launches.csv")))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum": continue
    n = r["Kernel Name"].split("(")[0].split("<")[0][-40:]
    agg[n][0] += 1; agg[n][1] += float(r["Metric Value"]) / 1e6
tot = sum(v[1] for v in agg.values())
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{n:42s} {c:5d} {t:9.3f} {100*t/tot:5.1f}%")
PY
