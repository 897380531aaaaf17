# GPU suite + C2 lines after the vectorised gradient-norm kernel.
timeout 900 python -m pytest tests -m gpu -q --tb=short -x 2>&1 | tail -2
for i in 1 2; do timeout 900 python bench.py --workload C2 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('C2', round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['clocks'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sqnorm --csv --log-file /tmp/sq.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python profiles/launch_summary.py /tmp/sq.csv | head -4
