# Timing variance of repeated cold solves, with SM clock / power samples alongside.
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv -lms 200 > gpurun_out/smi.csv &
SMI=$!
for i in 1 2; do
  ASG_REPS=5 ASG_EIGH_BATCH=64 timeout 900 python profiles/r01_phase.py eigh32 1024 2048 2>&1 | grep eigh32 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n'], [round(x) for x in d['reps']])"
  date +%T.%N
done
kill $SMI
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/smi.csv")))[1:]
import collections
print(len(rows), "samples")
for r in rows[::10]:
    print(",".join(x.strip() for x in r))
PY
