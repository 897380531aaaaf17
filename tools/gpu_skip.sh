# Rayleigh GEMM batch skip: GPU suite, then C2 bench lines.
timeout 900 python -m pytest tests -m gpu -q --tb=short -x 2>&1 | tail -2
for i in 1 2; do timeout 900 python bench.py --workload C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('C2', round(d['value'],1), 'ms', round(d['ms_per_step'],2), d['clocks'])"; done
ASG_EIGH_BATCH=64 ASG_REPS=3 timeout 600 python profiles/r01_phase.py eigh32 1024 2>&1 | grep eigh32 | cut -c1-200
