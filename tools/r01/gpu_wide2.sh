# Wide-pair threshold 768 (default) vs 256 for C2, interleaved; C5 n=512 both ways.
for cfg in "X=0" "ASG_TJ_WIDE_N=256" "X=0" "ASG_TJ_WIDE_N=256"; do
  env $cfg timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$cfg', round(d['value'],1), 'ms', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
for cfg in "X=0" "ASG_TJ_WIDE_N=256"; do
  env $cfg timeout 900 python bench.py --workload C5 --n 512 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('C5 512 $cfg', round(d['value'],3))"
done
