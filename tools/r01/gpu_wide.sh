# Wide-pair threshold: C5 cold points and C2 after kWidePairN = 768.
for cfg in "512 X=0" "512 ASG_TJ_WIDE_N=512" "1024 X=0" "1024 ASG_TJ_WIDE_N=4096"; do
  set -- $cfg
  env $2 timeout 900 python bench.py --workload C5 --n $1 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('C5 n=$1 $2', round(d['value'],3), 'ms', round(d['ms_per_step'],1))"
done
for i in 1 2; do timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('C2', round(d['value'],1), 'ms', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"; done
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --tb=short 2>&1 | tail -1
