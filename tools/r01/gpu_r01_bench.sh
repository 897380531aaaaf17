# GPU suite + smoke, then bench lines (TAG names the output set).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -3 > gpurun_out/r01_pytest_gpu_v${TAG}.log
cat gpurun_out/r01_pytest_gpu_v${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
for n in 1024 2048 4096 512; do
  timeout 1500 python bench.py --workload C5 --n $n --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_${n}_v${TAG}.jsonl 2>/tmp/c5_$n.err
done
for wl in C2 C3 C4 C1; do timeout 1200 python bench.py --workload $wl > gpurun_out/bench_${wl}_v${TAG}.jsonl 2>/tmp/$wl.err; done
for f in gpurun_out/bench_*_v${TAG}.jsonl; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], round(d['value'],4), 'ms', round(d['ms_per_step'],2), 'e2e', (d.get('e2e') or {}).get('value'), 'clk', d['clocks'], 'frac', (d.get('roofline') or {}).get('frac_of_mode_peak'))
"; done
