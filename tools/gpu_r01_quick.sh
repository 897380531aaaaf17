mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python profiles/r01_phase.py eigh 256 768 1024 2048 > gpurun_out/phase_eigh.jsonl 2>&1
timeout 900 python profiles/r01_phase.py step C2 C3 > gpurun_out/phase_step.jsonl 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/phase_eigh.jsonl gpurun_out/phase_step.jsonl
