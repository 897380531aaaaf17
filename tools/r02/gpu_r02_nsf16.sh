# NEWTON refresh with 3xFP16 iterates: root parity (small + 1024/2048), trajectories, smoke, C5 and C3 lines.
timeout 900 python -m pytest tests/test_gpu_newton.py -m gpu -q --tb=short -x 2>&1 | tail -4
timeout 1500 python -m pytest tests/test_gpu_parity_large.py -m gpu -q -s --tb=short -k "refresh_roots and 3 or c1_trajectory or c3_block" 2>&1 | grep -E "root errors|passed|failed|Error|assert" | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"], 2), round(d["ms_per_step"], 2), (d.get("step_ms") or {}).get("p50"), d["clocks"],
          (d.get("e2e") or {}).get("ms_per_step"), d.get("schedule"), d["config"].get("max_abs_XAX_minus_I"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
}
for n in 1024 2048; do
  for pr in 3xf16 3xtf32; do
    timeout 900 python bench.py --workload C5 --n $n --refresh newton --precision $pr --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ns_C5_${n}_$pr.jsonl 2>/dev/null; summ gpurun_out/r02_ns_C5_${n}_$pr.jsonl
  done
done
timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/r02_ns_C3.jsonl 2> gpurun_out/r02_ns_C3.err; summ gpurun_out/r02_ns_C3.jsonl
tail -2 gpurun_out/r02_ns_C3.err
