# C2 refresh diagnostics: phase timings and Jacobi sweep counts per refresh chunk.
mkdir -p gpurun_out
ASG_REFRESH_TIMING=1 ASG_TJ_REPORT=1 timeout 900 python bench.py --workload ${WL:-C2} --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c2diag.jsonl 2> gpurun_out/r02_c2diag.err
grep -E "refresh d=|sweeps|tj" gpurun_out/r02_c2diag.err | head -80
