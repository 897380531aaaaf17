# ncu --set full of the first C3 step's GEMMs (KL statistics: X = G R^-1 <2>, L <1>, Z^T <2>, R <1>; update <2>, APPLY <5>)
mkdir -p gpurun_out /tmp/ncu
ASG_NS_UNROLL=5 timeout -s KILL 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)(1|2|5)>" -s 0 -c 6 -o /tmp/ncu/c3_step \
  python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/c3_step.log 2>&1
python profiles/ncu_traffic.py /tmp/ncu/c3_step.ncu-rep > gpurun_out/r02_c3_ncu_full_step.txt 2>&1
cat gpurun_out/r02_c3_ncu_full_step.txt | head -20
cp /tmp/ncu/c3_step.ncu-rep gpurun_out/ 2>/dev/null
