# Batched C-ABI solvers on a cached scratch arena (chunked): parity + C5 lines.
timeout 900 python -m pytest tests/test_gpu_batched_solvers.py -m gpu -q --tb=short 2>&1 | tail -6
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    c = d["config"]
    print(sys.argv[1], round(d["value"], 2), round(d["ms_per_step"], 2), d["clocks"], c.get("max_abs_XAX_minus_I"), c.get("max_residual_rel"), d["dtype"][:40])
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
}
for n in 1024 2048; do
  for pr in 3xf16 3xtf32; do
    timeout 900 python bench.py --workload C5 --n $n --refresh newton --precision $pr --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ar_C5_${n}_$pr.jsonl 2>/dev/null; summ gpurun_out/r02_ar_C5_${n}_$pr.jsonl
  done
  timeout 900 python bench.py --workload C5 --n $n --refresh f32 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ar_C5_${n}_f32.jsonl 2>/dev/null; summ gpurun_out/r02_ar_C5_${n}_f32.jsonl
done
