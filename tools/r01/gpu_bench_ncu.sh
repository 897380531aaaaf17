# The ncu launch list of the bench command itself (C2, default workload), summarised.
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file /tmp/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/bench_ncu.log 2>&1
tail -1 /tmp/bench_ncu.log | cut -c1-200
python profiles/launch_summary.py /tmp/bench_launches.csv > gpurun_out/r01_bench_C2_ncu_launches.txt 2>&1
head -25 gpurun_out/r01_bench_C2_ncu_launches.txt
