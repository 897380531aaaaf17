# Timing experiment: the pair-tile GEMM issuing kind::f16 MMAs on the same staged bytes (half the K loop;
# numerics meaningless) against 3xTF32, short (unthrottled) and sustained (power-capped), with clocks.
for reps in 10 300; do
  for pr in 0 1; do
    nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 250 > /tmp/clk.txt & SMI=$!
    ASG_GEMM_BENCH_REPS=$reps ASG_GEMM_F16_PROBE=$pr python tools/r02/gemm_diag.py 0 2>&1 | grep bench
    kill $SMI; echo "probe $pr reps $reps clocks:"; sort /tmp/clk.txt | uniq -c | sort -rn | head -2
  done
done
ASG_GEMM_BENCH_REPS=10 python tools/r02/gemm_diag.py 2 2>&1 | grep bench
