echo "== debug sweeps (tol 1e-6), C2 warm refresh"
ASG_REFRESH=f32 ASG_EIGH_DEBUG=1 timeout 600 python profiles/r01_phase.py step C2 2>&1 | grep "tjdbg" | grep " b=0 " | tail -40
for tol in 3e-6 1e-5; do echo "== tol $tol"; ASG_F32_TOL=$tol ASG_REFRESH=f32 ASG_REFRESH_TIMING=1 timeout 600 python profiles/r01_phase.py step C2 2>&1 | tail -14 | cut -c1-200; done
