mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/pytest_gpu_all.log
ASG_EIGH_DEBUG=1 timeout 600 python -m pytest tests/test_gpu_multirank.py -q 2>&1 | tail -5 > gpurun_out/pytest_multirank_dbg.log
cat gpurun_out/pytest_gpu_all.log gpurun_out/pytest_multirank_dbg.log
