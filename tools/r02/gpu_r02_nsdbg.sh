# NEWTON iteration counts on the C3 factors (ASG_NS_DEBUG: per-iteration residuals).
ASG_NS_DEBUG=1 timeout 600 python bench.py --workload C3 --steps 1 --warmup 12 --no-e2e --no-cpu-baseline > /tmp/nsdbg.out 2>&1
grep nsdbg /tmp/nsdbg.out | awk '{print $2}' | sort | uniq -c | sort -k2 -t= -n | head -40
grep nsdbg /tmp/nsdbg.out | grep "b=0 " | head -40
