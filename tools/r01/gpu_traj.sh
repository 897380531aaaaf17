# F32 trajectory tests under the pair-solve variants (which one moves KL-Shampoo?).
for cfg in "X=0" "ASG_TJ_ROT32=0" "ASG_TJ_OE=0" "ASG_TJ_OE=0 ASG_TJ_ROT32=0"; do
  echo "== $cfg"
  env $cfg timeout -s KILL 600 python -m pytest tests/test_gpu_refresh_f32.py -q -k "bounded_staleness or rank_deficient or roots" --tb=line 2>&1 | grep -E "passed|failed|assert|Error" | cut -c1-300
done
