# ncu --set full of the C3 statistics product W = G P_R in both 3xTF32 storage modes
# (operand pairs in HBM: the default; plain fp32 split in shared memory: 3xtf32_smem);
# per-launch DRAM traffic into gpurun_out/r02_traffic.json (bench.py roofline.traffic).
mkdir -p gpurun_out /tmp/ncu
cp profiles/r02_traffic.json gpurun_out/r02_traffic.json
for pr in 3xtf32 3xtf32_smem; do  # (3xf16 below)
  spl=0; alg=25769803776; key=C3
  if [ $pr = 3xtf32_smem ]; then spl=1; alg=12884901888; key=C3_smem; fi
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)2, \(int\)2, \(bool\)$spl>" -s 3 -c 1 -o /tmp/ncu/w_$pr \
    python bench.py --workload C3 --precision $pr --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/w_$pr.log 2>&1
  python profiles/ncu_traffic.py /tmp/ncu/w_$pr.ncu-rep --json $key "gemm_tn_kernel<256, 3, 2, 2, $spl>" $alg gpurun_out/r02_traffic.json > gpurun_out/r02_c3_ncu_full_W_$pr.txt 2>&1
  cat gpurun_out/r02_c3_ncu_full_W_$pr.txt
  cp /tmp/ncu/w_$pr.ncu-rep gpurun_out/
done
# 3xFP16 (the bench default for C3): the W = G P_R product on fp16 pairs
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)2, \(int\)2, \(bool\)0, \(bool\)1>" -s 3 -c 1 -o /tmp/ncu/w_3xf16 \
  python bench.py --workload C3 --precision 3xf16 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/w_3xf16.log 2>&1
python profiles/ncu_traffic.py /tmp/ncu/w_3xf16.ncu-rep --json C3_f16 "gemm_tn_kernel<256, 3, 2, 2, 0, 1>" 12884901888 gpurun_out/r02_traffic.json > gpurun_out/r02_c3_ncu_full_W_3xf16.txt 2>&1
cat gpurun_out/r02_c3_ncu_full_W_3xf16.txt
cp /tmp/ncu/w_3xf16.ncu-rep gpurun_out/
