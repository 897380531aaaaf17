# Closing run of the last session: GPU suite + smoke on the tree with the faster tensor-core Jacobi,
# then bench lines C3 (default), C1, C2, C4, C5-F32 1024 / 2048.
mkdir -p gpurun_out
TAG=${TAG:-k}
timeout 1800 python -m pytest tests -m gpu -q --tb=short > gpurun_out/r02_pytest_gpu_${TAG}.log 2>&1
tail -3 gpurun_out/r02_pytest_gpu_${TAG}.log
grep -E "^FAILED" gpurun_out/r02_pytest_gpu_${TAG}.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"], 3), round(d.get("ms_per_step") or 0, 2), (d.get("step_ms") or {}).get("p50"),
          (d.get("clocks") or {}).get("sm_mhz"), (d.get("e2e") or {}).get("ms_per_step"), d.get("schedule"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
}
timeout 1200 python bench.py > gpurun_out/r02_${TAG}_default.jsonl 2> gpurun_out/r02_${TAG}_default.err; summ gpurun_out/r02_${TAG}_default.jsonl
for wl in C1 C2; do
  timeout 1200 python bench.py --workload $wl > gpurun_out/r02_${TAG}_$wl.jsonl 2>/dev/null; summ gpurun_out/r02_${TAG}_$wl.jsonl
done
timeout 1500 python bench.py --workload C4 --steps 12 --warmup 4 > gpurun_out/r02_${TAG}_C4.jsonl 2>/dev/null; summ gpurun_out/r02_${TAG}_C4.jsonl
for n in 1024 2048; do
  timeout 900 python bench.py --workload C5 --n $n --refresh f32 --steps 2 --warmup 1 > gpurun_out/r02_${TAG}_C5_${n}_f32.jsonl 2>/dev/null; summ gpurun_out/r02_${TAG}_C5_${n}_f32.jsonl
done
