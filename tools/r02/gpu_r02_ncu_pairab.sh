# DRAM traffic of the C3 W = G P_R GEMM with and without CTA pairs (ncu --set full, one launch each).
mkdir -p gpurun_out /tmp/ncu
for pr in 1 0; do
  if [ $pr = 1 ]; then rx='gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)2, \(int\)2>'; else rx='gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)2, \(int\)1>'; fi
  ASG_GEMM_PAIR=$pr timeout -s KILL 900 ncu --set full --clock-control none --kernel-name-base demangled \
    -k regex:"$rx" -s 3 -c 1 -o /tmp/ncu/pair$pr \
    python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/pair$pr.log 2>&1
  python profiles/ncu_traffic.py /tmp/ncu/pair$pr.ncu-rep 2>&1 | tail -2
  ncu -i /tmp/ncu/pair$pr.ncu-rep --page raw --csv --metrics lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum 2>/dev/null | tail -1 | cut -c1-400
done
