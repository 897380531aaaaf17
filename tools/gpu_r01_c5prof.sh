mkdir -p /tmp/ncu gpurun_out
ASG_EIGH_DEBUG=1 ASG_EIGH_BATCH=64 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file /tmp/ncu/c5.csv python profiles/r01_phase.py eigh32 2048 > /tmp/ncu/c5.log 2>&1
python profiles/launch_summary.py /tmp/ncu/c5.csv | head -12 > gpurun_out/r01_eigh32_2048_launches.txt; cat gpurun_out/r01_eigh32_2048_launches.txt
grep tjdbg /tmp/ncu/c5.log | grep " b=0 " | head -14
cuobjdump -sass paper_2605_16184_b200/csrc/build/asg_jacobi_tc.o | grep -E "Function|UTCHMMA|UTMALDG|UTCBAR|LDTM" | awk '{print $1, $2}' | sort | uniq -c | sort -rn | head -12 > gpurun_out/r01_tj_sass_summary.txt; cat gpurun_out/r01_tj_sass_summary.txt
