for env in "" "ASG_SIDE_SAME_PRIORITY=1" "ASG_NS_UNROLL=6"; do
  echo "== $env"
  env $env timeout 600 python bench.py --workload C3 --no-cpu-baseline --no-e2e --steps 14 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],1), d['step_ms']['per_step'])"
done
