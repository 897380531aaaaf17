mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload C2 > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.jsonl
timeout 900 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; cat gpurun_out/bench_c1.jsonl
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step1/" -k regex:gemm_tn_kernel -c 12 -o gpurun_out/c2_step_full python profiles/r01_steplaunch.py C2 1099511627776 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
