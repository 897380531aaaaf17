# Same-box A/B of the C3 step: tile raster order (ASG_GEMM_RASTER 0/1), interleaved, twice.
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), round(d["step_ms"]["p50"], 2), round(r["gemm_ms_per_step"], 2), d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
}
for i in 1 2; do
for ra in 0 1; do
ASG_GEMM_RASTER=$ra timeout 900 python bench.py --workload C3 --no-cpu-baseline --no-e2e > gpurun_out/r02_ra_${ra}_$i.jsonl 2>/dev/null; summ gpurun_out/r02_ra_${ra}_$i.jsonl
done
done
