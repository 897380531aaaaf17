# ncu --set full of the C3 step GEMMs (KL statistics EPI_SPLIT <2>, EPI_SYM_EMA <1>,
# update APPLY <5>) and the Newton-Schulz GEMMs (EPI_SYM_SPLIT <6>, EPI_NS <7>; the
# refresh runs unrolled, ASG_NS_UNROLL, so ncu sees plain launches).
mkdir -p gpurun_out /tmp/ncu
for sel in "1 2 5:-s 12 -c 3" "6 7:-s 4 -c 4"; do
  kinds=${sel%%:*}; opts=${sel#*:}; tag=$(echo $kinds | tr ' ' '_')
  re=$(echo $kinds | sed 's/ /|/g')
  ASG_NS_UNROLL=5 timeout -s KILL 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)($re)>" $opts -o /tmp/ncu/c3_full_$tag \
    python bench.py --workload C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/c3_full_$tag.log 2>&1
  tail -2 /tmp/ncu/c3_full_$tag.log | cut -c1-200
  python profiles/ncu_traffic.py /tmp/ncu/c3_full_$tag.ncu-rep > gpurun_out/r02_c3_ncu_full_$tag.txt 2>&1
  cat gpurun_out/r02_c3_ncu_full_$tag.txt | head -30
  cp /tmp/ncu/c3_full_$tag.ncu-rep gpurun_out/ 2>/dev/null
done
