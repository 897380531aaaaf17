# ncu --set full of the 3xFP16 C3 statistics products with fp16-pair epilogue outputs
# (W = G P_R, EPI_SPLIT; [V^T | V] = G^T P_L, EPI_SPLIT2) -> r02_traffic.json C3_f16;
# then C1 in both step arithmetics and the C3 3xTF32 storage modes on the current tree.
mkdir -p gpurun_out /tmp/ncu
cp profiles/r02_traffic.json gpurun_out/r02_traffic.json
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"gemm_tn_kernel<\(int\)256, \(int\)3, \(int\)(2|8), \(int\)2, \(bool\)0, \(bool\)1>" -s 6 -c 2 -o /tmp/ncu/w_f16out \
  python bench.py --workload C3 --precision 3xf16 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ncu/w_f16out.log 2>&1
python profiles/ncu_traffic.py /tmp/ncu/w_f16out.ncu-rep --json C3_f16 "gemm_tn_kernel<256, 3, 2, 2, 0, 1>" 12884901888 gpurun_out/r02_traffic.json > gpurun_out/r02_c3_ncu_full_f16out.txt 2>&1
cat gpurun_out/r02_c3_ncu_full_f16out.txt
cp /tmp/ncu/w_f16out.ncu-rep gpurun_out/
for cfg in "C1 3xf16" "C1 3xtf32" "C3 3xtf32" "C3 3xtf32_smem"; do
  set -- $cfg
  timeout 900 python bench.py --workload $1 --precision $2 --no-cpu-baseline > gpurun_out/r02_fx_$1_$2.jsonl 2> gpurun_out/r02_fx_$1_$2.err
  python - gpurun_out/r02_fx_$1_$2.jsonl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), d["step_ms"]["p50"], r["gemm_ms_per_step"], d["clocks"], d["e2e"]["ms_per_step"], d["schedule"]["barrier_waits"], d.get("state_bytes"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
