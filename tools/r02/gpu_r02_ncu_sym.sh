# ncu --set full of the C3 3xFP16 factor products (EPI_SYM_EMA, L and R) and the APPLY product.
mkdir -p /tmp/ncu
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)(1|5), \(int\)2, \(bool\)0, \(bool\)1>" -s 8 -c 3 -o /tmp/ncu/sym_f16 \
  python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/sym.log 2>&1
python profiles/ncu_traffic.py /tmp/ncu/sym_f16.ncu-rep > gpurun_out/r02_c3_ncu_full_sym_apply.txt 2>&1
cat gpurun_out/r02_c3_ncu_full_sym_apply.txt
cp /tmp/ncu/sym_f16.ncu-rep gpurun_out/
