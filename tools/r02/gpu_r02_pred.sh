# 3xFP16 gradient prep at the predicted scale (max fused, mispredicted blocks rewritten).
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_parity_large.py -m gpu -q --tb=short -k "f16 or operand_storage or 3 or trajectory" 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 3), d["step_ms"]["p50"], r["gemm_ms_per_step"], d["clocks"], d["e2e"]["ms_per_step"], d["schedule"], d["hbm_kernels"]["prep"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
}
for i in 1 2; do
timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/r02_pr_C3_$i.jsonl 2> gpurun_out/r02_pr_C3_$i.err; summ gpurun_out/r02_pr_C3_$i.jsonl
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_pr_launches.csv python bench.py --workload C3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/r02/launch_summary.py gpurun_out/r02_pr_launches.csv 20
