import ctypes as C, sys, json, torch
sys.path.insert(0, '.')
from paper_2605_16184_b200 import runtime as rt
res = []
for (b, M, N, K) in [(16, 2048, 2048, 2048), (64, 2048, 2048, 2048), (8, 1024, 1024, 1024), (16, 768, 1024, 768)]:
    for prec in (0, 1):
        A = torch.randn(b, M, K, device='cuda'); B = torch.randn(b, N, K, device='cuda'); Cm = torch.zeros(b, M, N, device='cuda')
        args = lambda: rt.check(rt.lib.asg_gemm_tn(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(Cm.data_ptr()), b, M, N, K, 1.0, 0.0, prec, None))
        for _ in range(3): args()
        torch.cuda.synchronize()
        # asg_gemm_tn includes the hi/lo split pre-pass; time end to end (split + GEMM)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); n = 5
        for _ in range(n): args()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        tf = 2 * b * M * N * K / ms / 1e9
        res.append(dict(batch=b, M=M, N=N, K=K, prec=['3xtf32', 'tf32'][prec], ms=ms, alg_tflops=tf))
        print(json.dumps(res[-1]), flush=True)
