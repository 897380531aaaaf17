# C2 with all step GEMMs at 128-wide tiles vs the default width rule, interleaved.
for cfg in "X=0" "ASG_GEMM_BN=128" "X=0" "ASG_GEMM_BN=128"; do
  env $cfg timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$cfg', round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'gemm ms/step', round(d['roofline']['gemm_ms_per_step'],2), d['clocks']['sm_mhz'])"
done
