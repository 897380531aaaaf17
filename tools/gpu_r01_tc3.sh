mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
ASG_EIGH_BATCH=64 timeout 900 python profiles/r01_phase.py eigh32 256 512 1024 2048 4096 2>&1 | tail -5
ASG_REFRESH=f32 timeout 900 python profiles/r01_phase.py step C2 C3 2>&1 | tail -4
timeout 900 python bench.py --workload C2 --no-cpu-baseline 2>gpurun_out/bench_c2.err | tee gpurun_out/bench_c2.jsonl
timeout 900 python bench.py --workload C3 --no-cpu-baseline 2>gpurun_out/bench_c3.err | tee gpurun_out/bench_c3.jsonl
