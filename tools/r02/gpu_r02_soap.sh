# SOAP workloads with fresh gradients (F32 tensor-core Jacobi refresh) + split-API / full GPU suite
mkdir -p gpurun_out
for wl in C2 C4; do
  timeout 1500 python bench.py --workload $wl --no-cpu-baseline --steps 20 > gpurun_out/r02_bench_${wl}_${TAG}.jsonl 2> gpurun_out/r02_bench_${wl}_${TAG}.err
  python -c "
import json; d=json.loads(open('gpurun_out/r02_bench_${wl}_${TAG}.jsonl').readline())
print('$wl', round(d['value'],2), 'ms', round(d['ms_per_step'],2), d['step_ms']['per_step'], d['schedule'])"
done
