timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
ASG_EIGH_BATCH=64 timeout 900 python profiles/r01_phase.py eigh32 256 1024 2048 2>&1 | tail -3
ASG_REFRESH=f32 ASG_REFRESH_TIMING=1 timeout 600 python profiles/r01_phase.py step C2 2>&1 | tail -14 | cut -c1-200
for wl in C1 C2 C3; do timeout 900 python bench.py --workload $wl --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print(d['config']['workload'][:30], 'value', round(d['value'],2), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],2), 'launches', d['gpu_launches'], 'gemm_ms', round(d['roofline']['gemm_ms_per_step'],2))"; done
