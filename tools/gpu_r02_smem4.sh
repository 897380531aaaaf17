python tools/gemm_diag.py 0
for dg in 0 1 2 3; do ASG_GEMM_DIAG=$dg python tools/gemm_diag.py 2; done
ASG_GEMM_SPL_DUAL=0 python tools/gemm_diag.py 2
