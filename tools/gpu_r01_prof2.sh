mkdir -p gpurun_out
NCU="ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx"
ASG_EIGH_DEBUG=0 timeout 900 $NCU --nvtx-include "step1/" --log-file gpurun_out/c2_step_launches.csv python profiles/r01_steplaunch.py C2 1099511627776 2 > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/c2_step_launches.csv > gpurun_out/c2_step_sum.txt; head -14 gpurun_out/c2_step_sum.txt
timeout 900 $NCU --nvtx-include "step1/" --log-file gpurun_out/c3_step_launches.csv python profiles/r01_steplaunch.py C3 1099511627776 2 > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/c3_step_launches.csv > gpurun_out/c3_step_sum.txt; head -12 gpurun_out/c3_step_sum.txt
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step1/" -k regex:gemm_tn_kernel -o gpurun_out/c2_gemm_full python profiles/r01_steplaunch.py C2 1099511627776 2 > gpurun_out/ncu_c2full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step1/" -k regex:gemm_tn_kernel -o gpurun_out/c3_gemm_full python profiles/r01_steplaunch.py C3 1099511627776 2 > gpurun_out/ncu_c3full.log 2>&1
tail -2 gpurun_out/ncu_c2full.log gpurun_out/ncu_c3full.log
