mkdir -p /tmp/ncu
ASG_EIGH_DEBUG=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx --nvtx-include "step2/" -c 400 --log-file /tmp/ncu/w.csv python profiles/r01_steplaunch.py C2 1 3 > /dev/null 2>&1
python - <<'PY'
import sys
sys.path.insert(0, 'profiles')
import launch_summary as L
ls = L.load('/tmp/ncu/w.csv')
for i, (n, us) in enumerate(ls[:140]):
    short = n.split('(')[0].replace('void ', '').replace('asg::<unnamed>::', '')[:40]
    print(i, short, round(us, 1))
PY
