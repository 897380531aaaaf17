# Launch list of one warm synchronous C2 refresh step (pf=1; step 2), plain launches (debug).
mkdir -p gpurun_out
ASG_EIGH_DEBUG=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step2/" --csv --log-file /tmp/c2r.csv python profiles/r01_steplaunch.py C2 1 3 > /tmp/c2r.log 2>&1
tail -2 /tmp/c2r.log
python profiles/launch_summary.py /tmp/c2r.csv > gpurun_out/r01_c2_refresh_warm_v9_launches.txt 2>&1
head -30 gpurun_out/r01_c2_refresh_warm_v9_launches.txt
