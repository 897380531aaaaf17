mkdir -p gpurun_out
ASG_EIGH_DEBUG=1 ASG_EIGH_BATCH=64 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/eigh32_2048_launches.csv python profiles/r01_phase.py eigh32 2048 > gpurun_out/eigh32_dbg.log 2>&1
grep tjdbg gpurun_out/eigh32_dbg.log | grep "b=0 " | head -20
python profiles/launch_summary.py gpurun_out/eigh32_2048_launches.csv > gpurun_out/eigh32_sum.txt; head -12 gpurun_out/eigh32_sum.txt
