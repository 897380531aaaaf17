# Kernel-only timing of the 3xTF32 GEMM modes on a C3-shaped batched product:
# asg_gemm_tn with ASG_GEMM_REPEAT = 1 and 11 (same operands); the difference
# / 10 is one GEMM launch. Environment knobs select kernel variants.
import ctypes as C, os, subprocess, sys, time  # run from the repo root: python tools/r02/gemm_diag.py PREC
sys.path.insert(0, os.getcwd())
if len(sys.argv) > 2:  # child: time one configuration
    import torch
    from paper_2605_16184_b200 import runtime as rt
    b, n = 64, 2048
    A = torch.randn(b, n, n, device="cuda"); B = torch.randn(b, n, n, device="cuda"); Cm = torch.zeros(b, n, n, device="cuda")
    prec = int(sys.argv[1])
    def run():
        rt.check(rt.lib.asg_gemm_tn(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(Cm.data_ptr()), b, n, n, n, 1.0, 0.0, prec, None))
    run(); torch.cuda.synchronize()
    t = []
    for _ in range(3):
        t0 = time.perf_counter(); run(); torch.cuda.synchronize(); t.append(time.perf_counter() - t0)
    print(min(t))
    sys.exit(0)
prec = sys.argv[1]
res = {}
for k in (1, 11):
    env = dict(os.environ, ASG_GEMM_REPEAT=str(k))
    res[k] = float(subprocess.run([sys.executable, __file__, prec, "child"], env=env, capture_output=True, text=True).stdout.strip().splitlines()[-1])
ms = (res[11] - res[1]) / 10 * 1e3
print(f"prec {prec} diag {os.environ.get('ASG_GEMM_DIAG', '0')} dual {os.environ.get('ASG_GEMM_SPL_DUAL', '1')}: "
      f"{ms:.2f} ms per GEMM ({2 * 64 * 2048 ** 3 / ms / 1e9:.0f} TFLOP/s)")
