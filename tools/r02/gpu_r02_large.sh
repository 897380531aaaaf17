# Round 2: large-n parity tests (wide-pair Jacobi, bench-size refreshes, C1/C3 trajectories) + Newton-Schulz roots.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_newton.py tests/test_gpu_parity_large.py -m gpu -q -s --tb=short > gpurun_out/r02_pytest_large.log 2>&1
grep -E "matrix|root errors|SOAP|trajectory|passed|failed|FAILED|Error|error" gpurun_out/r02_pytest_large.log | tail -90
