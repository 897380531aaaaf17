# Full GPU suite + smoke + the default bench lines (TAG names the logs).
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 1500 python -m pytest tests -m gpu -q --tb=short > gpurun_out/r02_pytest_gpu_${TAG}.log 2>&1
tail -15 gpurun_out/r02_pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -4
for wl in ${WORKLOADS:-C3 C1}; do
  timeout 1200 python bench.py --workload $wl > gpurun_out/r02_bench_${wl}_${TAG}.jsonl 2> gpurun_out/r02_bench_${wl}_${TAG}.err
  echo "== $wl rc=$?"; tail -c 1500 gpurun_out/r02_bench_${wl}_${TAG}.jsonl; tail -3 gpurun_out/r02_bench_${wl}_${TAG}.err
done
