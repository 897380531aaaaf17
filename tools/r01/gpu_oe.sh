# Cold tensor-core Jacobi timing A/B over pair-solve variants (min of 3 solves).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_refresh_f32.py -q -x --tb=short 2>&1 | tail -2
run() { env "$@" ASG_EIGH_BATCH=64 timeout 900 python profiles/r01_phase.py eigh32 $N 2>&1 | grep eigh32 | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$N $*', round(d['ms_per_matrix'],3), 'ms/matrix', [round(x) for x in d['reps']], 'res', '%.1e'%d['residual'], 'orth', '%.1e'%d['orth'])"; }
N=2048
run X=0; run ASG_TJ_OE=0; run ASG_TJ_NT=1024; run ASG_TJ_ROT32=1; run ASG_TJ_NT=1024 ASG_TJ_ROT32=1
N=1024
run X=0; run ASG_TJ_WIDE_N=1024; run ASG_TJ_WIDE_N=1024 ASG_TJ_NT=1024 ASG_TJ_ROT32=1; run ASG_TJ_ROT32=1 ASG_TJ_OE=1
N=512
run X=0; run ASG_TJ_WIDE_N=512 ASG_TJ_ROT32=1
