# Warm-refresh cost in C2 (phase timings + sweeps), parity, and C2 lines.
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_refresh_f32.py -q -x --tb=short 2>&1 | tail -1
ASG_TJ_REPORT=1 ASG_REFRESH_TIMING=1 timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e --steps 20 > /tmp/c2.json 2> /tmp/c2.err
grep "^refresh" /tmp/c2.err | tail -11 | awk '{for(i=1;i<=NF;i++) if($i=="eigh") e+=$(i+1); else if ($i=="transform") t+=$(i+1)} END {print "last refresh cycle: transform", t, "ms, eigh", e, "ms"}'
for i in 1 2; do timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('C2', round(d['value'],1), 'ms', round(d['ms_per_step'],2), d['clocks'])"; done
