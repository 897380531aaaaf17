mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
ASG_REFRESH=f32 timeout 900 python profiles/r01_phase.py step C2 C3 > gpurun_out/phase_step_f32.jsonl 2>&1
cat gpurun_out/phase_step_f32.jsonl
timeout 900 python bench.py --workload C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.jsonl; tail -5 gpurun_out/bench_c2.err
