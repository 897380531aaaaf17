# ncu launch list of the default bench command (C3) at the closing state.
mkdir -p gpurun_out /tmp/ncu
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file /tmp/ncu/c3f.csv \
  python bench.py --steps 2 --warmup 8 --no-e2e --no-cpu-baseline > /tmp/ncu/c3f.log 2>&1
python profiles/launch_summary.py /tmp/ncu/c3f.csv > gpurun_out/r02_bench_C3_ncu_launches_final.txt 2>&1
head -30 gpurun_out/r02_bench_C3_ncu_launches_final.txt
