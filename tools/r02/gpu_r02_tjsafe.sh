# Warm eigensolve timings + eigen/F32-refresh parity, every step under its own timeout (kernel changes
# with new mbarrier protocols: a deadlock must end the process, not the box).
mkdir -p gpurun_out
ASG_TJ_REPORT=1 timeout 180 python tools/r02/tj_warm.py 1024 64 3 > gpurun_out/tj_time_1024_${TAG}.log 2>&1; echo "rc=$?"; grep -v tjreport gpurun_out/tj_time_1024_${TAG}.log | tail -3
ASG_TJ_REPORT=1 timeout 180 python tools/r02/tj_warm.py 2048 32 3 > gpurun_out/tj_time_2048_${TAG}.log 2>&1; echo "rc=$?"; grep -v tjreport gpurun_out/tj_time_2048_${TAG}.log | tail -3
timeout 900 python -m pytest -x -q tests/test_gpu_kernels.py tests/test_gpu_parity_large.py tests/test_gpu_refresh_f32.py > gpurun_out/pytest_tjsym_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_tjsym_${TAG}.log
