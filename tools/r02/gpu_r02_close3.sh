# Final check after the adaptive gradient-norm chunks: GPU suite + smoke, C1 and the default (C3) line.
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 1800 python -m pytest tests -m gpu -q --tb=short > gpurun_out/r02_pytest_gpu_${TAG}.log 2>&1
tail -2 gpurun_out/r02_pytest_gpu_${TAG}.log
grep -E "^FAILED" gpurun_out/r02_pytest_gpu_${TAG}.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
for wl in C1 C3; do
  timeout 1200 python bench.py --workload $wl > gpurun_out/r02_${TAG}_$wl.jsonl 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r02_${TAG}_$wl.jsonl').read().strip().splitlines()[-1])
print('$wl', round(d['value'],2), round(d['ms_per_step'],3), d['step_ms']['p50'], d['clocks'], d['e2e']['ms_per_step'], d['schedule'], d.get('hbm_kernels'))"
done
