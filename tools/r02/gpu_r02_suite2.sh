# Full GPU suite + smoke + C1 / C3 lines (128-wide symmetric tiles for few-matrix groups).
timeout 3000 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r02_pytest_gpu_s2.log
cat gpurun_out/r02_pytest_gpu_s2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 3), d["step_ms"]["p50"], r["gemm_ms_per_step"], d["clocks"], d["e2e"]["ms_per_step"], d["schedule"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
}
timeout 900 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/r02_s2_C1.jsonl 2> gpurun_out/r02_s2_C1.err; summ gpurun_out/r02_s2_C1.jsonl
ASG_GEMM_BN=0 timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/r02_s2_C3.jsonl 2> gpurun_out/r02_s2_C3.err; summ gpurun_out/r02_s2_C3.jsonl
