# SOAP-refresh bench lines after the eigensolver changes: C2, C4 (fresh gradients, F32 Jacobi refresh), C5 F32 at 1024 / 2048.
mkdir -p gpurun_out
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
timeout 900 python bench.py --workload C2 > gpurun_out/r02_tj_C2_${TAG}.jsonl 2>gpurun_out/r02_tj_C2_${TAG}.err; summ gpurun_out/r02_tj_C2_${TAG}.jsonl
for n in 1024 2048; do
  timeout 900 python bench.py --workload C5 --n $n --refresh f32 --steps 2 --warmup 1 > gpurun_out/r02_tj_C5_${n}_f32_${TAG}.jsonl 2>/dev/null; summ gpurun_out/r02_tj_C5_${n}_f32_${TAG}.jsonl
done
timeout 1500 python bench.py --workload C4 --steps 12 --warmup 4 > gpurun_out/r02_tj_C4_${TAG}.jsonl 2>/dev/null; summ gpurun_out/r02_tj_C4_${TAG}.jsonl
