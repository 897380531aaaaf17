# Round-2 baseline: GPU suite, smoke, quick bench lines C2/C3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -5 > gpurun_out/r02_pytest_gpu_base.log
cat gpurun_out/r02_pytest_gpu_base.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
for wl in C2 C3; do timeout 900 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/r02_bench_${wl}_base.jsonl 2>gpurun_out/r02_bench_${wl}_base.err; tail -c 600 gpurun_out/r02_bench_${wl}_base.jsonl; done
