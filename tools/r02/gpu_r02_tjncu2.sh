# Timings of the current pair/apply kernels + one early-sweep ncu --set full of the pair kernel.
mkdir -p gpurun_out
ASG_TJ_REPORT=1 python tools/r02/tj_warm.py 1024 64 3 > gpurun_out/tj_time_1024_${TAG}.log 2>&1; grep -v tjreport gpurun_out/tj_time_1024_${TAG}.log | tail -3
ASG_TJ_REPORT=1 python tools/r02/tj_warm.py 2048 32 3 > gpurun_out/tj_time_2048_${TAG}.log 2>&1; grep -v tjreport gpurun_out/tj_time_2048_${TAG}.log | tail -3
ASG_EIGH_DEBUG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tj_pair_kernel -s 3 -c 1 -o gpurun_out/tj_pair_${TAG} python tools/r02/tj_warm.py 2048 32 > gpurun_out/ncu_pair.log 2>&1; tail -1 gpurun_out/ncu_pair.log
