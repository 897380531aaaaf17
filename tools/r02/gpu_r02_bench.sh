# Round-2 bench lines (fresh gradients every step). TAG names the set; WORKLOADS / EXTRA override.
mkdir -p gpurun_out
for wl in ${WORKLOADS:-C3 C1}; do
  timeout 1200 python bench.py --workload $wl ${EXTRA:-} > gpurun_out/r02_bench_${wl}_${TAG}.jsonl 2> gpurun_out/r02_bench_${wl}_${TAG}.err
  echo "== $wl rc=$?"; tail -c 3000 gpurun_out/r02_bench_${wl}_${TAG}.jsonl; tail -3 gpurun_out/r02_bench_${wl}_${TAG}.err
done
