# KL reformulation follow-up: large parity tests, C3 bench, C2 with / without CTA pairs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_newton.py tests/test_gpu_precond.py tests/test_gpu_split_api.py -m gpu -q --tb=short 2>&1 | tail -4
timeout 900 python bench.py --workload C3 > gpurun_out/r02_kl2_C3.jsonl 2> gpurun_out/r02_kl2_C3.err
for pr in 1 0; do
  ASG_GEMM_PAIR=$pr timeout 900 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/r02_kl2_C2_pair$pr.jsonl 2> gpurun_out/r02_kl2_C2_pair$pr.err
done
python - <<'PY'
import json
for f in ["gpurun_out/r02_kl2_C3.jsonl","gpurun_out/r02_kl2_C2_pair1.jsonl","gpurun_out/r02_kl2_C2_pair0.jsonl"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"],1), round(d["ms_per_step"],2), d["step_ms"]["p50"], round(d["roofline"]["frac_of_mode_peak"],3), round(d["roofline"]["gemm_ms_per_step"],2), d["clocks"], d["state_bytes"]/1e9, d.get("workspace_bytes",0)/1e9, d["e2e"]["ms_per_step"])
    except Exception as e: print(f, "ERR", e)
PY
