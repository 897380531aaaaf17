mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
for inner in 4 2 1; do echo "inner=$inner"; ASG_TJ_INNER=$inner ASG_EIGH_BATCH=64 timeout 600 python profiles/r01_phase.py eigh32 1024 2048 2>&1 | tail -2; done
ASG_REFRESH=f32 timeout 900 python profiles/r01_phase.py step C2 C3 2>&1 | tail -4
timeout 900 python bench.py --workload C3 --steps 20 --no-cpu-baseline 2>gpurun_out/bench_c3.err | tee gpurun_out/bench_c3.jsonl
