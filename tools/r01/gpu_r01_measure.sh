set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python profiles/r01_phase.py eigh 256 512 768 1024 2048 > gpurun_out/phase_eigh.jsonl 2>&1
timeout 900 python profiles/r01_phase.py step C2 C3 > gpurun_out/phase_step.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/eigh1024_launches.csv python profiles/r01_phase.py eigh 1024 > gpurun_out/ncu_eigh.log 2>&1
tail -3 gpurun_out/*.log gpurun_out/*.jsonl
