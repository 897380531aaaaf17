# A/B on one box: 3xFP16 gradient prep with the predicted scale (ASG_F16_PRED=1) vs max pass + prep (0).
timeout 900 python -m pytest tests/test_gpu_step.py -m gpu -q --tb=short -k "f16 or operand_storage" 2>&1 | tail -2
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 3), d["step_ms"]["p50"], round(r["gemm_ms_per_step"], 2), d["clocks"]["sm_mhz"], round(d["hbm_kernels"]["prep"]["ms_per_step"], 2), round(d["synth_ms_per_step"], 2))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
}
for i in 1 2; do
for pr in 1 0; do
ASG_F16_PRED=$pr timeout 900 python bench.py --workload C3 --no-cpu-baseline --no-e2e > gpurun_out/r02_p3_C3_${pr}_$i.jsonl 2>/dev/null; summ gpurun_out/r02_p3_C3_${pr}_$i.jsonl
done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:prep -c 40 --csv --log-file gpurun_out/r02_p3_launches.csv python bench.py --workload C3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -E "prep" gpurun_out/r02_p3_launches.csv | awk -F'","' '{print $5" | "$9" | "$15}' | cut -c1-30,150- | head -12
