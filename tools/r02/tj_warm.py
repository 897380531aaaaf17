# Warm-refresh-like F32 eigensolve: B = Q^T (0.6 A1 + 0.4 A_fresh) Q with Q the
# eigenbasis of A1 (what a SOAP refresh solves with fresh gradients, pf 10, beta 0.95).
import ctypes as C, os, sys, time
import torch
sys.path.insert(0, os.getcwd())
from paper_2605_16184_b200 import runtime as rt
n, b = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
torch.manual_seed(0)
def spd():
    x = torch.randn(b, n, 2 * n, device='cuda')
    return torch.baddbmm(1e-3 * torch.eye(n, device='cuda').expand(b, n, n), x, x.transpose(1, 2), alpha=1.0 / (2 * n))
a1 = spd()
_, q = torch.linalg.eigh(a1.double())
a2 = 0.6 * a1 + 0.4 * spd()
bm = (q.transpose(1, 2) @ a2.double() @ q).float().contiguous()
bm = 0.5 * (bm + bm.transpose(1, 2))
w = torch.empty(b, n, dtype=torch.float64, device='cuda'); v = torch.empty(b, n, n, device='cuda')
for r in range(reps):
    torch.cuda.synchronize(); t = time.perf_counter()
    rt.check(rt.lib.asg_sym_eig_batched_f32(C.c_void_p(bm.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(v.data_ptr()), b, n, None))
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f'n={n} b={b} rep={r} {dt*1e3:.1f} ms ({dt*1e3/b:.2f} ms/factor)')
wd = w.double(); vd = v.double()
res = (bm.double() @ vd - vd * wd[:, None, :]).norm(dim=(1, 2)) / bm.double().norm(dim=(1, 2))
orth = (vd.transpose(1, 2) @ vd - torch.eye(n, device='cuda', dtype=torch.float64)).norm(dim=(1, 2))
ref = torch.linalg.eigvalsh(bm.double())
print('resid max', res.max().item(), 'orth max', orth.max().item(), 'eig relerr', ((wd - ref).abs().max() / ref.abs().max()).item())
