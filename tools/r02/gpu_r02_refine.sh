# NEWTON refinement only for long product chains: Newton parity tests, large roots / trajectories, C3 bench.
timeout 900 python -m pytest tests/test_gpu_newton.py tests/test_gpu_parity_large.py -m gpu -q -s --tb=short -k "newton or NEWTON or roots or trajectory" 2>&1 | grep -E "root errors|trajectory|passed|failed|FAIL" | tail -30
timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/r02_refine_C3.jsonl 2>/dev/null
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_refine_C3.jsonl").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["step_ms"]["p50"], d["step_ms"]["per_step"], d["roofline"]["gemm_ms_per_step"], d["clocks"], d["schedule"])
PY
