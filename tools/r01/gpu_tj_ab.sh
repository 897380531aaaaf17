# Serialised pair-kernel time (ncu launch list) of the odd-even pair solves; NS="..." picks sizes.
mkdir -p gpurun_out
for n in ${NS:-2048 1024 512}; do
  ASG_EIGH_DEBUG=1 ASG_EIGH_BATCH=64 ASG_REPS=1 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tj_pair --csv --log-file /tmp/l.csv python profiles/r01_phase.py eigh32 $n > /tmp/o.txt 2>&1
  python profiles/launch_summary.py /tmp/l.csv > /tmp/s.txt 2>&1; echo "$n: $(sed -n 3p /tmp/s.txt)  $(grep -o '"residual": [0-9.e-]*' /tmp/o.txt)"
done
