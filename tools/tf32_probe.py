import sys, os; sys.path.insert(0, os.getcwd())
import ctypes as C, torch
from paper_2605_16184_b200 import runtime as rt
M=N=128; K=32
for frac in (0.25, 0.5, 0.75):
    x = 1.0 + frac * 2.0**-10
    A = torch.full((1, M, K), x, dtype=torch.float32, device="cuda")
    B = torch.ones((1, N, K), dtype=torch.float32, device="cuda")
    Cm = torch.zeros((1, M, N), dtype=torch.float32, device="cuda")
    rt.check(rt.lib.asg_gemm_tn(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(Cm.data_ptr()), 1, M, N, K, 1.0, 0.0, 1, None))
    torch.cuda.synchronize()
    v = Cm[0,0,0].item() / K
    print(f"x = 1 + {frac} ulp_tf32: tensor core used {v!r} -> ({(v-1)/2**-10:.3f} ulp)")
