# Narrow (64-wide) vs wide (128-wide) Jacobi pairs under fresh-gradient (cold-like) refreshes:
# C5 solves at n = 1024 / 2048 and the C2 bench, ASG_TJ_WIDE_N = 512 (default) vs 4096 (narrow everywhere).
for wn in 512 4096; do
  for n in 1024 2048; do
    ASG_TJ_WIDE_N=$wn timeout 900 python bench.py --workload C5 --n $n --refresh f32 --steps 2 --warmup 1 > /tmp/w.jsonl 2>/dev/null
    python - $wn $n <<'PY'
import json, sys
d = json.loads(open("/tmp/w.jsonl").read().strip().splitlines()[-1])
print("wide_n", sys.argv[1], "n", sys.argv[2], round(d["ms_per_step"], 1), "ms per solve", round(d["value"], 2), "TF/s")
PY
  done
  ASG_TJ_WIDE_N=$wn timeout 900 python bench.py --workload C2 --no-cpu-baseline > /tmp/c2.jsonl 2>/dev/null
  python - $wn <<'PY'
import json, sys
d = json.loads(open("/tmp/c2.jsonl").read().strip().splitlines()[-1])
print("wide_n", sys.argv[1], "C2", round(d["ms_per_step"], 2), d["step_ms"]["p50"], d["schedule"])
PY
done
