mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k f32 2>&1 | tail -5
ASG_EIGH_BATCH=16 timeout 600 python profiles/r01_phase.py eigh32 256 512 1024 2048 2>&1 | tail -8
