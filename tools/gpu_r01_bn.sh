python profiles/r01_gemm_microbench.py 2>&1 | tail -8
ASG_GEMM_BN=128 python profiles/r01_gemm_microbench.py 2>&1 | tail -8
