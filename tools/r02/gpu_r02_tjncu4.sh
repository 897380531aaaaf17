# ncu --set full of one early-sweep pair solve on the final tree (sweeps unrolled), warm 2048^2 x 32.
mkdir -p gpurun_out
ASG_EIGH_DEBUG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tj_pair_kernel -s 3 -c 1 -o gpurun_out/tj_pair_${TAG} python tools/r02/tj_warm.py 2048 32 > gpurun_out/ncu_pair.log 2>&1; tail -1 gpurun_out/ncu_pair.log
