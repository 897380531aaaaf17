mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/r01_pytest_gpu_v5.log
for wl in C2 C1 C3 C4; do timeout 1200 python bench.py --workload $wl > gpurun_out/bench_$wl.jsonl 2> /tmp/ncu/bench_$wl.err; done
timeout 1200 python bench.py --workload C5 --n 2048 --steps 2 --warmup 3 > gpurun_out/bench_C5_2048.jsonl 2> /tmp/ncu/c5.err
timeout 1200 python bench.py --workload C5 --n 1024 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_1024.jsonl 2> /tmp/ncu/c5b.err
timeout 600 python bench.py --workload C2 --impl reference > gpurun_out/bench_C2_ref.jsonl 2>/dev/null
timeout 600 python bench.py --workload C1 --impl reference > gpurun_out/bench_C1_ref.jsonl 2>/dev/null
cat gpurun_out/r01_pytest_gpu_v5.log
for f in gpurun_out/bench_*.jsonl; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], d.get('impl','ours'), 'value', round(d['value'],4), 'ms', round(d['ms_per_step'],2), 'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'frac', (d.get('roofline') or {}).get('frac'))
"; done
