# A/B of the wide pair solve's thread count (ASG_TJ_NT 512 / 1024) on the warm eigensolve, same box.
mkdir -p gpurun_out
for nt in 512 1024 512; do
  ASG_TJ_NT=$nt python tools/r02/tj_warm.py 2048 32 3 2>&1 | tail -2 | head -1 | sed "s/^/NT=$nt /"
  ASG_TJ_NT=$nt python tools/r02/tj_warm.py 1024 64 3 2>&1 | tail -2 | head -1 | sed "s/^/NT=$nt /"
done
