set -x
mkdir -p gpurun_out
NCU="ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx"
timeout 900 $NCU --nvtx-include "step1/" --log-file gpurun_out/c3_step_launches.csv python profiles/r01_steplaunch.py C3 1099511627776 2 > gpurun_out/c3_step.log 2>&1
timeout 900 $NCU --nvtx-include "step1/" --log-file gpurun_out/c2_step_launches.csv python profiles/r01_steplaunch.py C2 1099511627776 2 > gpurun_out/c2_step.log 2>&1
timeout 1200 $NCU --nvtx-include "step2/" -c 60000 --log-file gpurun_out/c2_refresh_launches.csv python profiles/r01_steplaunch.py C2 1 3 > gpurun_out/c2_refresh.log 2>&1
for f in gpurun_out/c3_step_launches.csv gpurun_out/c2_step_launches.csv gpurun_out/c2_refresh_launches.csv; do python profiles/launch_summary.py $f | head -30; done
