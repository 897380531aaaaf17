# GPU test suite + quick bench lines (no CPU baseline) for C2 / C3 / C4.
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
for wl in ${WORKLOADS:-C2 C3 C4}; do timeout 900 python bench.py --workload $wl --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print(d['config']['workload'][:30], 'value', round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],2), 'roof', round(d['roofline']['achieved'],1), round(d['roofline']['frac_of_mode_peak'],3))"; done
