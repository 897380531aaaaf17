# Final round-1 bench lines + the ncu capture behind roofline.traffic.
mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/r01_pytest_gpu_v6.log
for wl in C2 C1 C3 C4; do timeout 1200 python bench.py --workload $wl > gpurun_out/bench_$wl.jsonl 2> /tmp/ncu/bench_$wl.err; done
timeout 1200 python bench.py --workload C5 --n 2048 --steps 2 --warmup 3 > gpurun_out/bench_C5_2048.jsonl 2> /tmp/ncu/c5.err
timeout 1200 python bench.py --workload C5 --n 1024 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_1024.jsonl 2> /tmp/ncu/c5b.err
for wl in C2 C1 C3; do timeout 600 python bench.py --workload $wl --impl reference > gpurun_out/bench_${wl}_ref.jsonl 2>/dev/null; done
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step1/" -k regex:gemm_tn_kernel -c 3 -o /tmp/ncu/c3_full python profiles/r01_steplaunch.py C3 1099511627776 2 > /tmp/ncu/c3full.log 2>&1
python profiles/ncu_traffic.py /tmp/ncu/c3_full.ncu-rep --json C3 "gemm_tn_kernel<256, 3, 2>" 25769803776 gpurun_out/r01_traffic_c3.json > gpurun_out/r01_c3_gemm_ncu_full_v6.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step1/" -k regex:gemm_tn_kernel -c 12 -o /tmp/ncu/c2_full python profiles/r01_steplaunch.py C2 1099511627776 2 > /tmp/ncu/c2full.log 2>&1
python profiles/ncu_traffic.py /tmp/ncu/c2_full.ncu-rep > gpurun_out/r01_c2_gemm_ncu_full_v6.txt 2>&1
cat gpurun_out/r01_pytest_gpu_v6.log gpurun_out/r01_c3_gemm_ncu_full_v6.txt gpurun_out/r01_c2_gemm_ncu_full_v6.txt
for f in gpurun_out/bench_*.jsonl; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], d.get('impl','ours'), 'value', round(d['value'],4), 'ms', round(d['ms_per_step'],2), 'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'frac', (d.get('roofline') or {}).get('frac'))
"; done
