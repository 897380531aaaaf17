# 3xFP16 step chains (Shampoo / KL-Shampoo): GEMM + trajectory parity, then C3 / C1 bench against 3xTF32.
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q --tb=short -k gemm 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_parity_large.py -m gpu -q -s --tb=short -k trajectory 2>&1 | grep -E "trajectory|passed|failed|Error" | tail -16
for wl in C3 C1; do
  for pr in 3xf16 3xtf32; do
    timeout 900 python bench.py --workload $wl --precision $pr --no-cpu-baseline > gpurun_out/r02_f16_${wl}_$pr.jsonl 2> gpurun_out/r02_f16_${wl}_$pr.err
    python - gpurun_out/r02_f16_${wl}_$pr.jsonl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), d["step_ms"]["p50"], r["gemm_ms_per_step"], d["clocks"], round(d["state_bytes"] / 1e9, 1), d["e2e"]["ms_per_step"], d["schedule"]["barrier_waits"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
    tail -2 gpurun_out/r02_f16_${wl}_$pr.err
  done
done
