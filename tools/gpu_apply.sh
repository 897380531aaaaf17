# Sweeps per solve in graph mode (is the timing variance borderline convergence?) + per-kernel apply time.
mkdir -p gpurun_out
ASG_TJ_REPORT=1 ASG_REPS=8 ASG_EIGH_BATCH=64 timeout -s KILL 900 python profiles/r01_phase.py eigh32 512 1024 2048 2>&1 | grep -E "tjreport|eigh32" | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['n'], round(d['ms_per_matrix'],3), 'ms/matrix', [round(x) for x in d['reps']])
    else: print(l.strip())"
