# In-smem split with the dual ring (SPL = 2): GEMM tests + trajectories, C3/C2 A/B vs pairs-in-HBM, dual on/off.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --tb=short -k gemm 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_parity_large.py -m gpu -q --tb=short -k "trajectory" 2>&1 | tail -3
for wl in C3 C2; do
  for cfg in "3xtf32_smem 1" "3xtf32 1" "3xtf32_smem 0"; do
    set -- $cfg
    ASG_GEMM_SPL_DUAL=$2 timeout 900 python bench.py --workload $wl --precision $1 --no-cpu-baseline > gpurun_out/r02_smem3_${wl}_$1_$2.jsonl 2> gpurun_out/r02_smem3_${wl}_$1_$2.err
    python - gpurun_out/r02_smem3_${wl}_$1_$2.jsonl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), d["step_ms"]["p50"], r["gemm_ms_per_step"], d["clocks"], d["state_bytes"] / 1e9, d["e2e"]["ms_per_step"])
PY
  done
done
