# Parity, then serialised pair-kernel time (ncu launch list) for the batched odd-even pass.
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_refresh_f32.py -q -x --tb=short 2>&1 | tail -2
for nc in "2048 X=0" "2048 ASG_TJ_ROT32=1" "1024 X=0" "1024 ASG_TJ_OE=1" "512 X=0" "512 ASG_TJ_OE=1"; do
  set -- $nc
  n=$1; shift
  env "$@" ASG_EIGH_DEBUG=1 ASG_EIGH_BATCH=64 ASG_REPS=1 timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tj_pair --csv --log-file /tmp/l.csv python profiles/r01_phase.py eigh32 $n > /tmp/o.txt 2>&1
  python profiles/launch_summary.py /tmp/l.csv > /tmp/s.txt 2>&1; echo "$n $*: $(sed -n 3p /tmp/s.txt)  $(grep -o '"residual": [0-9.e-]*' /tmp/o.txt)"
done
