# C2 bench with refresh phase timings and per-solve sweep counts (stderr diagnostics).
ASG_TJ_REPORT=1 ASG_REFRESH_TIMING=1 timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e --steps 20 > /tmp/c2.json 2> /tmp/c2.err
python -c "
import json; d=json.loads(open('/tmp/c2.json').readline()); print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],2))"
grep -c tjreport /tmp/c2.err
grep tjreport /tmp/c2.err | sort | uniq -c | sort -rn | head -20
grep "^refresh" /tmp/c2.err | tail -12
