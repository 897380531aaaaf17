# Where a cold F32 eigensolve's time goes at n = 1024 (C2's block size): serialised ncu launch list of
# one C5 solve with the sweeps unrolled (ASG_EIGH_DEBUG; 128 factors).
mkdir -p gpurun_out /tmp/ncu
ASG_EIGH_DEBUG=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file /tmp/ncu/tj.csv \
  python -c "
import ctypes as C, sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2605_16184_b200 import runtime as rt
n, b = 1024, 128
x = torch.randn(b, n, 2 * n, device='cuda')
a = torch.baddbmm(1e-3 * torch.eye(n, device='cuda').expand(b, n, n), x, x.transpose(1, 2), alpha=1.0 / (2 * n))
w = torch.empty(b, n, dtype=torch.float64, device='cuda'); v = torch.empty(b, n, n, device='cuda')
rt.check(rt.lib.asg_sym_eig_batched_f32(C.c_void_p(a.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(v.data_ptr()), b, n, None))
torch.cuda.synchronize(); print('ok')
" > /tmp/ncu/tj.log 2>&1
tail -2 /tmp/ncu/tj.log
python profiles/launch_summary.py /tmp/ncu/tj.csv > gpurun_out/r02_tj_n1024_launches.txt 2>&1
head -16 gpurun_out/r02_tj_n1024_launches.txt
