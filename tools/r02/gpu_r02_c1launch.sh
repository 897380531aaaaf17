# C1 (one 1024^2 Shampoo block, NEWTON refresh every step): serialised launch list of 3 steps.
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file /tmp/ncu/c1.csv \
  python bench.py --workload C1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/c1.log 2>&1
python profiles/launch_summary.py /tmp/ncu/c1.csv > gpurun_out/r02_c1_launches.txt 2>&1
head -30 gpurun_out/r02_c1_launches.txt
