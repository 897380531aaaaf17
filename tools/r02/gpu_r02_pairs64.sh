# C3 with the pair-tile grid capped at 64 pairs (one batch of 8 x 8 tiles per wave; 20 SMs left to the
# side-stream refresh) vs the full 74: step time, GEMM time, clocks; then the W launch's DRAM traffic.
for cap in 0 64; do
  ASG_GEMM_MAX_PAIRS=$cap timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/r02_pairs${cap}_C3.jsonl 2>/dev/null
  python - gpurun_out/r02_pairs${cap}_C3.jsonl $cap <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("cap", sys.argv[2], round(d["ms_per_step"], 2), d["step_ms"]["p50"], round(d["roofline"]["gemm_ms_per_step"], 2), d["clocks"], d["step_ms"]["per_step"][:6])
PY
done
mkdir -p /tmp/ncu
ASG_GEMM_MAX_PAIRS=64 timeout -s KILL 900 ncu --set full --clock-control none --kernel-name-base demangled \
  -k regex:'gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)2, \(int\)2, \(bool\)0>' -s 3 -c 1 -o /tmp/ncu/p64 \
  python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/p64.log 2>&1
python profiles/ncu_traffic.py /tmp/ncu/p64.ncu-rep 2>&1 | tail -1
