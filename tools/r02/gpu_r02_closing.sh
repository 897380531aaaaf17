# Round-2 closing run on the final tree: GPU suite + smoke, the default bench line (C3 + CPU
# baseline) and the reference arm as the driver runs them, C1/C2/C4/C5 lines, the launch list.
mkdir -p gpurun_out /tmp/ncu
TAG=${TAG:-g}
timeout 2400 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/r02_pytest_gpu_${TAG}.log 2>&1
tail -3 gpurun_out/r02_pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    print(sys.argv[1], round(d["value"], 3), round(d.get("ms_per_step") or 0, 2), (d.get("step_ms") or {}).get("p50"),
          r.get("gemm_ms_per_step"), r.get("frac_of_mode_peak"), d.get("clocks"), e.get("ms_per_step"),
          (d.get("schedule") or {}).get("barrier_waits"), (d.get("state_bytes") or 0) / 1e9, (d.get("cpu_baseline") or {}).get("value"))
except Exception as ex:
    print(sys.argv[1], "ERR", ex)
PY
}
timeout 1200 python bench.py > gpurun_out/r02_${TAG}_default.jsonl 2> gpurun_out/r02_${TAG}_default.err; summ gpurun_out/r02_${TAG}_default.jsonl
timeout 1200 python bench.py --impl reference > gpurun_out/r02_${TAG}_reference.jsonl 2> gpurun_out/r02_${TAG}_reference.err; summ gpurun_out/r02_${TAG}_reference.jsonl
timeout 1200 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/r02_${TAG}_C3_b.jsonl 2>/dev/null; summ gpurun_out/r02_${TAG}_C3_b.jsonl
timeout 900 python bench.py --workload C1 > gpurun_out/r02_${TAG}_C1.jsonl 2>/dev/null; summ gpurun_out/r02_${TAG}_C1.jsonl
timeout 900 python bench.py --workload C2 > gpurun_out/r02_${TAG}_C2.jsonl 2>/dev/null; summ gpurun_out/r02_${TAG}_C2.jsonl
timeout 1500 python bench.py --workload C4 --steps 12 --warmup 4 --no-cpu-baseline > gpurun_out/r02_${TAG}_C4.jsonl 2>/dev/null; summ gpurun_out/r02_${TAG}_C4.jsonl
for rf in newton f32; do
  timeout 900 python bench.py --workload C5 --n 2048 --refresh $rf --steps 2 --warmup 1 > gpurun_out/r02_${TAG}_C5_2048_$rf.jsonl 2>/dev/null; summ gpurun_out/r02_${TAG}_C5_2048_$rf.jsonl
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file /tmp/ncu/c3final.csv \
  python bench.py --steps 2 --warmup 8 --no-e2e --no-cpu-baseline > /tmp/ncu/c3final.log 2>&1
python tools/r02/launch_summary.py /tmp/ncu/c3final.csv 30 > gpurun_out/r02_bench_C3_ncu_launches_${TAG}.txt 2>&1
head -16 gpurun_out/r02_bench_C3_ncu_launches_${TAG}.txt
