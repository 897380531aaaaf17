# Warm F32 eigensolve: timings (no profiler), then a serialised launch list with the
# sweeps unrolled (ASG_EIGH_DEBUG) and one ncu --set full of the pair and apply kernels at 2048.
mkdir -p gpurun_out /tmp/ncu
ASG_TJ_REPORT=1 python tools/r02/tj_warm.py 1024 64 3 > gpurun_out/tj_time_1024.log 2>&1; tail -5 gpurun_out/tj_time_1024.log
ASG_TJ_REPORT=1 python tools/r02/tj_warm.py 2048 32 3 > gpurun_out/tj_time_2048.log 2>&1; tail -5 gpurun_out/tj_time_2048.log
ASG_EIGH_DEBUG=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file /tmp/ncu/tj2048.csv \
  python tools/r02/tj_warm.py 2048 16 > /tmp/ncu/tj.log 2>&1
python profiles/launch_summary.py /tmp/ncu/tj2048.csv > gpurun_out/r02_tj_warm2048_launches.txt 2>&1
head -16 gpurun_out/r02_tj_warm2048_launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tj_pair_kernel -s 40 -c 1 -o gpurun_out/tj_pair python tools/r02/tj_warm.py 2048 32 > /tmp/ncu/p.log 2>&1; tail -2 /tmp/ncu/p.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tj_apply_kernel -s 40 -c 1 -o gpurun_out/tj_apply python tools/r02/tj_warm.py 2048 32 > /tmp/ncu/a.log 2>&1; tail -2 /tmp/ncu/a.log
