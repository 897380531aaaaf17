# Two refresh side streams (own workspace sets): GPU suite, then same-box A/B (ASG_REFRESH_STREAMS 1/2) on C2, C3, C4.
timeout 2400 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/r02_pytest_gpu_st.log 2>&1
tail -3 gpurun_out/r02_pytest_gpu_st.log
grep -E "^FAILED|Error" gpurun_out/r02_pytest_gpu_st.log | head -10
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["value"], 2), round(d["ms_per_step"], 2), round(d["step_ms"]["p50"], 2), d["clocks"]["sm_mhz"], d["schedule"]["barrier_waits"], round(d["schedule"]["barrier_wait_ms"], 1), round(d["workspace_bytes"] / 1e9, 1))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
}
for wl in C2 C3; do
for ns in 2 1; do
ASG_REFRESH_STREAMS=$ns timeout 900 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/r02_st_${wl}_$ns.jsonl 2>/dev/null; summ gpurun_out/r02_st_${wl}_$ns.jsonl
done
done
for ns in 2 1; do
ASG_REFRESH_STREAMS=$ns timeout 1500 python bench.py --workload C4 --steps 12 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/r02_st_C4_$ns.jsonl 2>/dev/null; summ gpurun_out/r02_st_C4_$ns.jsonl
done
