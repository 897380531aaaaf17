# DRAM traffic of the C3 W = G P_R pair GEMM under two tile rasters (ncu --set full, one launch each).
mkdir -p gpurun_out /tmp/ncu
for ra in 0 1; do
  ASG_GEMM_RASTER=$ra timeout -s KILL 900 ncu --set full --clock-control none --kernel-name-base demangled \
    -k regex:'gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)2, \(int\)2>' -s 3 -c 1 -o /tmp/ncu/ra$ra \
    python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/ra$ra.log 2>&1
  python profiles/ncu_traffic.py /tmp/ncu/ra$ra.ncu-rep 2>&1 | tail -1
  ncu -i /tmp/ncu/ra$ra.ncu-rep --page raw --csv --metrics lts__t_sector_hit_rate.pct 2>/dev/null | tail -1 | rev | cut -d, -f1 | rev
done
