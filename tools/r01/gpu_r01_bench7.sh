# GPU suite, then bench lines after the odd-even pair solves (C5 at 1024/2048/4096, C3/C4 warm refresh).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -3 > gpurun_out/r01_pytest_gpu_v7.log
cat gpurun_out/r01_pytest_gpu_v7.log
for n in 2048 1024 4096; do
  timeout 1500 python bench.py --workload C5 --n $n --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_${n}_v7.jsonl 2>/tmp/c5_$n.err
done
for wl in C3 C4 C2; do timeout 1200 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/bench_${wl}_v7.jsonl 2>/tmp/$wl.err; done
for f in gpurun_out/bench_*_v7.jsonl; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],4), 'ms', round(d['ms_per_step'],2), 'e2e', (d.get('e2e') or {}).get('value'), 'clk', d['clocks'])
"; done
