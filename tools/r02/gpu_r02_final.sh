# Round-2 closing run: GPU suite + smoke, then the bench lines (C3 twice, C1, C2) and the C3 reference arm.
mkdir -p gpurun_out
TAG=${TAG:-f}
timeout 1500 python -m pytest tests -m gpu -q --tb=short > gpurun_out/r02_pytest_gpu_${TAG}.log 2>&1
tail -3 gpurun_out/r02_pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
for run in "C3 a" "C3 b" "C1 a" "C2 a"; do
  set -- $run
  timeout 1200 python bench.py --workload $1 > gpurun_out/r02_${TAG}_$1_$2.jsonl 2> gpurun_out/r02_${TAG}_$1_$2.err
  python - gpurun_out/r02_${TAG}_$1_$2.jsonl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(sys.argv[1], round(d["value"], 2), round(d["ms_per_step"], 2), d["step_ms"]["p50"], r.get("gemm_ms_per_step"), r.get("frac_of_mode_peak"), d["clocks"], d["e2e"]["ms_per_step"], d["schedule"], d["state_bytes"] / 1e9)
PY
done
timeout 900 python bench.py --workload C3 --impl reference --steps 3 --warmup 1 > gpurun_out/r02_${TAG}_C3_reference.jsonl 2>&1; tail -c 300 gpurun_out/r02_${TAG}_C3_reference.jsonl
bash tools/r02/gpu_r02_ncu_traffic.sh 2>&1 | grep -E "gemm_tn|wrote" | cut -c1-200
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file /tmp/ncu/c3final.csv \
  python bench.py --steps 2 --warmup 8 --no-e2e --no-cpu-baseline > /tmp/ncu/c3final.log 2>&1
python profiles/launch_summary.py /tmp/ncu/c3final.csv > gpurun_out/r02_bench_C3_ncu_launches_${TAG}.txt 2>&1
head -14 gpurun_out/r02_bench_C3_ncu_launches_${TAG}.txt
