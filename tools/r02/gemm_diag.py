# Kernel-only timing of the tensor-core GEMM on a C3-shaped batch (64 x 2048^3) through the
# diagnostics entry asg_gemm_tn with ASG_GEMM_BENCH_REPS (CUDA events over prepared operands).
# Usage (repo root): ASG_GEMM_BENCH_REPS=200 python tools/r02/gemm_diag.py PREC
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2605_16184_b200 import runtime as rt
b, n = 64, 2048
A = torch.randn(b, n, n, device="cuda"); B = torch.randn(b, n, n, device="cuda"); Cm = torch.zeros(b, n, n, device="cuda")
rt.check(rt.lib.asg_gemm_tn(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(Cm.data_ptr()), b, n, n, n,
                            1.0, 0.0, int(sys.argv[1]), None))
