# 3xFP16 GEMM: accuracy against fp64 (test_gemm_tn_matches_fp64[3-...]) and kernel time against 3xTF32.
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q --tb=short -k gemm 2>&1 | tail -4
for pr in 0 3 2; do ASG_GEMM_BENCH_REPS=200 python tools/r02/gemm_diag.py $pr 2>&1 | grep bench | sed "s/^/prec $pr: /"; done
