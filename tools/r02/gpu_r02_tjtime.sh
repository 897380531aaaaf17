# Warm eigensolve timings only (A/B of pair-kernel variants), each under a timeout.
mkdir -p gpurun_out
ASG_TJ_REPORT=1 timeout 180 python tools/r02/tj_warm.py 1024 64 3 > gpurun_out/tj_time_1024_${TAG}.log 2>&1; grep -v tjreport gpurun_out/tj_time_1024_${TAG}.log | tail -2
ASG_TJ_REPORT=1 timeout 180 python tools/r02/tj_warm.py 2048 32 3 > gpurun_out/tj_time_2048_${TAG}.log 2>&1; grep -v tjreport gpurun_out/tj_time_2048_${TAG}.log | tail -2
