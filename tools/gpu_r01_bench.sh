mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
for wl in C2 C1 C3 C4; do timeout 1200 python bench.py --workload $wl > gpurun_out/bench_$wl.jsonl 2> gpurun_out/bench_$wl.err; tail -c 300 gpurun_out/bench_$wl.err; done
timeout 900 python bench.py --workload C5 --n 1024 --steps 2 --warmup 3 > gpurun_out/bench_C5_1024.jsonl 2> gpurun_out/bench_C5.err
timeout 900 python bench.py --workload C2 --impl reference > gpurun_out/bench_C2_ref.jsonl 2>> gpurun_out/bench_C5.err
for f in gpurun_out/bench_*.jsonl; do echo $f; python -c "
import json,sys
for l in open('$f'):
    d=json.loads(l); print(d.get('impl','ours'), d['config'].get('workload','')[:40], 'value', round(d['value'],3), 'ms', round(d['ms_per_step'],2), 'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'frac', (d.get('roofline') or {}).get('frac'))
"; done
