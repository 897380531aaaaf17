# C2 with the narrow pair ordering A/B (odd-even default vs round-robin), interleaved.
for cfg in "X=0" "ASG_TJ_OE=0" "X=0" "ASG_TJ_OE=0"; do
  env $cfg timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$cfg', round(d['value'],1), 'ms', round(d['ms_per_step'],2), d['clocks'], 'gemm ms/step', round(d['roofline']['gemm_ms_per_step'],2))"
done
