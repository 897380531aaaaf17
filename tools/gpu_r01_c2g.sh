mkdir -p /tmp/ncu
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --nvtx --nvtx-include "step1/" -k regex:gemm_tn_kernel --log-file /tmp/ncu/c2g.csv python profiles/r01_steplaunch.py C2 1099511627776 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('/tmp/ncu/c2g.csv')))
start = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[start]
ki, mi, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
idi = hdr.index('ID')
by = {}
for r in rows[start+1:]:
    if len(r) <= vi: continue
    d = by.setdefault(r[idi], {'k': r[ki].split('(')[0].replace('void ','')})
    d[r[mi]] = (r[vi], r[ui])
for i, d in by.items():
    print(i, d['k'], {k.split('__')[1][:25]: v for k, v in d.items() if k != 'k'})
PY
