# In-smem split, lo-only converter: GEMM tests + C3/C2 A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --tb=short -k gemm 2>&1 | tail -3
for wl in C3 C2; do
  for pr in 3xtf32_smem 3xtf32; do
    timeout 900 python bench.py --workload $wl --precision $pr --no-cpu-baseline > gpurun_out/r02_smem2_${wl}_$pr.jsonl 2> gpurun_out/r02_smem2_${wl}_$pr.err
    python - gpurun_out/r02_smem2_${wl}_$pr.jsonl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), d["step_ms"]["p50"], r["gemm_ms_per_step"], d["clocks"], d["state_bytes"] / 1e9, d["e2e"]["ms_per_step"])
PY
  done
done
