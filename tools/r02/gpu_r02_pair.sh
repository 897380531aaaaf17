# CTA-pair GEMM: kernel tests, then C3 bench with and without pairs.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --tb=short -k gemm 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_precond.py tests/test_gpu_newton.py -m gpu -q -x --tb=short 2>&1 | tail -5
for pr in 1 0; do
  ASG_GEMM_PAIR=$pr timeout 900 python bench.py --workload ${WL:-C3} > gpurun_out/r02_pair${pr}_${WL:-C3}.jsonl 2> gpurun_out/r02_pair${pr}.err
  echo "== pair=$pr rc=$?"; python - <<PY
import json
d=json.loads(open("gpurun_out/r02_pair${pr}_${WL:-C3}.jsonl").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["step_ms"]["p50"], d["roofline"]["frac_of_mode_peak"], d["roofline"]["gemm_ms_per_step"], d["clocks"])
PY
  tail -2 gpurun_out/r02_pair${pr}.err
done
