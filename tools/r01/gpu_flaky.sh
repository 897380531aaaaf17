# Repeat the whole GPU suite with failure tracebacks (diagnosing an
# order-dependent failure); keeps the log of every run that fails.
mkdir -p gpurun_out
for i in 1 2 3 4 5; do
  timeout 900 python -m pytest tests -m gpu -q --tb=long -rf -p no:randomly > /tmp/pf_$i.log 2>&1
  tail -1 /tmp/pf_$i.log
  if grep -q FAILED /tmp/pf_$i.log; then cp /tmp/pf_$i.log gpurun_out/pytest_flaky_$i.log; fi
done
