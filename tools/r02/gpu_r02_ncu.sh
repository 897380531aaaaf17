# Round 2 profiles: (1) ncu launch list of the C3 bench command itself (fresh
# gradients, Newton refresh; graph kernel nodes listed individually);
# (2) ncu --set full of the dominant step GEMM (KL statistics EPI_SPLIT),
# the update APPLY GEMM and the Newton-Schulz EPI_NS / EPI_SYM_SPLIT GEMMs.
mkdir -p gpurun_out /tmp/ncu
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file /tmp/ncu/c3_launches.csv \
  python bench.py --workload C3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/c3_bench.log 2>&1
tail -c 300 /tmp/ncu/c3_bench.log
python profiles/launch_summary.py /tmp/ncu/c3_launches.csv > gpurun_out/r02_bench_C3_ncu_launches.txt 2>&1
head -30 gpurun_out/r02_bench_C3_ncu_launches.txt
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm_tn_kernel<256, 3, (2|5|6|7)>" -s 30 -c 6 -o /tmp/ncu/c3_full \
  python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/c3_full.log 2>&1
tail -3 /tmp/ncu/c3_full.log
python profiles/ncu_traffic.py /tmp/ncu/c3_full.ncu-rep > gpurun_out/r02_c3_ncu_full.txt 2>&1
cat gpurun_out/r02_c3_ncu_full.txt | head -40
cp /tmp/ncu/c3_full.ncu-rep gpurun_out/ 2>/dev/null
