# Wide pairs from n=768 (fewer rounds per sweep) for the C2 warm refresh: A/B.
for cfg in "X=0" "ASG_TJ_WIDE_N=768"; do
  env $cfg ASG_REFRESH_TIMING=1 timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e --steps 20 > /tmp/c2.json 2> /tmp/c2.err
  echo "$cfg $(grep '^refresh' /tmp/c2.err | tail -11 | awk '{for(i=1;i<=NF;i++) if($i=="eigh") e+=$(i+1); else if ($i=="transform") t+=$(i+1)} END {print "transform", t, "eigh", e}')"
  for i in 1 2; do env $cfg timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('  C2', round(d['value'],1), 'ms', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"; done
done
ASG_TJ_WIDE_N=768 ASG_EIGH_BATCH=64 ASG_REPS=3 timeout 600 python profiles/r01_phase.py eigh32 1024 2>&1 | grep eigh32 | cut -c1-150
ASG_EIGH_BATCH=64 ASG_REPS=3 timeout 600 python profiles/r01_phase.py eigh32 1024 2>&1 | grep eigh32 | cut -c1-150
