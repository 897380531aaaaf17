# Round-2 C3 profiles after the KL reformulation + CTA-pair GEMMs: (1) ncu
# launch list of the bench command; (2) ncu --set full of the step's pair GEMMs
# (W = G P_R EPI_SPLIT <2>, V^T/V EPI_SPLIT2 <8>, statistics EPI_SYM_EMA <1>,
# update EPI_APPLY <5>) -> traffic per launch (profiles/r02_traffic.json).
mkdir -p gpurun_out /tmp/ncu
if [ -z "$SKIP_LIST" ]; then
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file /tmp/ncu/c3_launches.csv \
  python bench.py --workload C3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/c3_bench.log 2>&1
python profiles/launch_summary.py /tmp/ncu/c3_launches.csv > gpurun_out/r02_bench_C3_ncu_launches_kl.txt 2>&1
head -24 gpurun_out/r02_bench_C3_ncu_launches_kl.txt
fi
timeout -s KILL 1800 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)(1|2|5|8), \(int\)2>" -s 20 -c 6 -o /tmp/ncu/c3_full_kl \
  python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/c3_full_kl.log 2>&1
tail -2 /tmp/ncu/c3_full_kl.log | cut -c1-300
cp profiles/r01_traffic.json gpurun_out/r02_traffic.json
python profiles/ncu_traffic.py /tmp/ncu/c3_full_kl.ncu-rep --json C3 "gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)2, \(int\)2>" 25769803776 gpurun_out/r02_traffic.json > gpurun_out/r02_c3_ncu_full_kl.txt 2>&1
cat gpurun_out/r02_c3_ncu_full_kl.txt | head -30
cp /tmp/ncu/c3_full_kl.ncu-rep gpurun_out/ 2>/dev/null
