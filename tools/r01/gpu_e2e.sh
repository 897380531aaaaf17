# e2e with one flat pinned gradient batch per step.
for wl in C2 C3; do timeout 900 python bench.py --workload $wl --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$wl', round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2), 'h2d', d['e2e']['h2d_bytes_per_step'])"; done
