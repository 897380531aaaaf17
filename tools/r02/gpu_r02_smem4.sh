# Kernel-only GEMM timing of the two 3xTF32 storage modes (tools/r02/gemm_diag.py).
python tools/r02/gemm_diag.py 0
python tools/r02/gemm_diag.py 2
