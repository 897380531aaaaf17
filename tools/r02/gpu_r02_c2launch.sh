# ncu launch list of a C2 bench run across refresh steps: where the SOAP refresh time goes (pair vs apply).
mkdir -p gpurun_out /tmp/ncu
ASG_TJ_REPORT=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/ncu/c2_launches.csv \
  python bench.py --workload C2 --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/c2_bench.log 2>&1
python profiles/launch_summary.py /tmp/ncu/c2_launches.csv > gpurun_out/r02_bench_C2_ncu_launches.txt 2>&1
head -30 gpurun_out/r02_bench_C2_ncu_launches.txt
