# fp16-pair epilogue outputs at a bound-derived scale (no to_f16pair passes), T16/S16 aliasing, absmax grids.
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_precond.py -m gpu -q --tb=short -x 2>&1 | tail -4
timeout 1500 python -m pytest tests/test_gpu_parity_large.py -m gpu -q -s --tb=short -k "trajectory" 2>&1 | grep -E "passed|failed|Error|assert" | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/r02_fo_C3.jsonl 2> gpurun_out/r02_fo_C3.err
timeout 900 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/r02_fo_C1.jsonl 2> gpurun_out/r02_fo_C1.err
for f in gpurun_out/r02_fo_C3.jsonl gpurun_out/r02_fo_C1.jsonl; do
python - $f <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), d["step_ms"]["p50"], r["gemm_ms_per_step"], d["clocks"], d["e2e"]["ms_per_step"], d["schedule"]["barrier_waits"], d.get("state_bytes"), d.get("workspace_bytes"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
tail -2 gpurun_out/r02_fo_C3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_fo_launches.csv python bench.py --workload C3 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo ncu rc $?
