# ncu --set full of the C3 W = G P_R GEMM in the in-smem split mode (one launch).
mkdir -p gpurun_out /tmp/ncu
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:'gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)2, \(int\)2, \(bool\)1>' -s 3 -c 1 -o /tmp/ncu/smem \
  python bench.py --workload C3 --precision 3xtf32_smem --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/smem.log 2>&1
tail -2 /tmp/ncu/smem.log | cut -c1-200
python profiles/ncu_traffic.py /tmp/ncu/smem.ncu-rep 2>&1 | tail -2
ncu -i /tmp/ncu/smem.ncu-rep --page details --csv 2>/dev/null | grep -E "Shared|smsp__pcsamp|Stall|Warp Cycles|Issue|Bank|L1/TEX|Tensor|Throughput" | head -60 > gpurun_out/r02_ncu_smem_details.txt
cat gpurun_out/r02_ncu_smem_details.txt | cut -c1-220 | head -60
cp /tmp/ncu/smem.ncu-rep gpurun_out/
