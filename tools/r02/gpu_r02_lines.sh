# Round-2 bench lines: C3 with / without CTA pairs (same box), C2, C4, C5 (f32 eigensolve and NEWTON roots).
mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d.get("roofline", {})
print(sys.argv[1], round(d["value"], 3), round(d.get("ms_per_step") or 0, 2), (d.get("step_ms") or {}).get("p50"),
      r.get("frac_of_mode_peak"), r.get("gemm_ms_per_step"), d.get("clocks"), (d.get("e2e") or {}).get("ms_per_step"),
      d.get("schedule"))
PY
}
for pr in 1 0; do
  ASG_GEMM_PAIR=$pr timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/r02_lines_C3_pair$pr.jsonl 2>/dev/null; summ gpurun_out/r02_lines_C3_pair$pr.jsonl
done
timeout 900 python bench.py --workload C2 > gpurun_out/r02_lines_C2.jsonl 2>/dev/null; summ gpurun_out/r02_lines_C2.jsonl
timeout 1500 python bench.py --workload C4 --steps 12 --warmup 4 > gpurun_out/r02_lines_C4.jsonl 2>/dev/null; summ gpurun_out/r02_lines_C4.jsonl
for n in 1024 2048; do
  for rf in f32 newton; do
    timeout 900 python bench.py --workload C5 --n $n --refresh $rf --steps 2 --warmup 1 > gpurun_out/r02_lines_C5_${n}_$rf.jsonl 2>/dev/null; summ gpurun_out/r02_lines_C5_${n}_$rf.jsonl
  done
done
