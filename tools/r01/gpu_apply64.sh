# 64B-swizzled 4-deep MMA1 ring in the Jacobi apply: bounded parity first, then serialised apply time.
mkdir -p gpurun_out
timeout -s KILL 240 python profiles/r01_phase.py eigh32 512 2>&1 | grep -E "eigh32|rror" | cut -c1-220
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_refresh_f32.py -q -x --tb=short 2>&1 | tail -2
for n in 2048; do
  ASG_EIGH_DEBUG=1 ASG_EIGH_BATCH=16 ASG_REPS=3 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tj_apply --csv --log-file /tmp/l.csv python profiles/r01_phase.py eigh32 $n > /tmp/o.txt 2>&1
  python profiles/launch_summary.py /tmp/l.csv > /tmp/s.txt 2>&1; echo "$n: $(sed -n 3p /tmp/s.txt)  $(grep -o '"residual": [0-9.e-]*' /tmp/o.txt)"
done
