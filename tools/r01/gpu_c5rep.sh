# C5 n=2048 spread over repeated runs (with sweep reports).
for i in 1 2 3; do ASG_TJ_REPORT=1 timeout 900 python bench.py --workload C5 --n 2048 --steps 2 --warmup 3 --no-cpu-baseline 2>/tmp/e.txt | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('C5 2048', round(d['value'],3), 'ms', round(d['ms_per_step'],1))"; grep tjreport /tmp/e.txt | sort | uniq -c | head -4; done
