# ncu --set full of one early-sweep pair solve and one apply (sweeps unrolled by ASG_EIGH_DEBUG so
# the kernels launch outside the CUDA graph), warm 2048^2 factors.
mkdir -p gpurun_out
ASG_EIGH_DEBUG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tj_pair_kernel -s 3 -c 1 -o gpurun_out/tj_pair python tools/r02/tj_warm.py 2048 32 > gpurun_out/ncu_pair.log 2>&1; tail -2 gpurun_out/ncu_pair.log
ASG_EIGH_DEBUG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tj_apply_kernel -s 3 -c 1 -o gpurun_out/tj_apply python tools/r02/tj_warm.py 2048 32 > gpurun_out/ncu_apply.log 2>&1; tail -2 gpurun_out/ncu_apply.log
ls -la gpurun_out
