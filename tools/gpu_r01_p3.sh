mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
ASG_EIGH_BATCH=64 timeout 900 python profiles/r01_phase.py eigh32 256 512 1024 2048 4096 2>&1 | tail -5
NCU="ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx"
ASG_EIGH_DEBUG=1 timeout 900 $NCU --nvtx-include "step2/" -c 20000 --log-file /tmp/ncu/c2_refresh.csv python profiles/r01_steplaunch.py C2 1 3 > /dev/null 2>&1
python profiles/launch_summary.py /tmp/ncu/c2_refresh.csv > gpurun_out/r01_c2_refresh_f32_launches.txt; head -22 gpurun_out/r01_c2_refresh_f32_launches.txt
timeout 600 $NCU --nvtx-include "step1/" --log-file /tmp/ncu/c2s.csv python profiles/r01_steplaunch.py C2 1099511627776 2 > /dev/null 2>&1
python profiles/launch_summary.py /tmp/ncu/c2s.csv > gpurun_out/r01_c2_step_launches.txt; head -12 gpurun_out/r01_c2_step_launches.txt
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step1/" -k regex:gemm_tn_kernel -c 3 -o /tmp/ncu/c3_full python profiles/r01_steplaunch.py C3 1099511627776 2 > /tmp/ncu/c3full.log 2>&1
python profiles/ncu_traffic.py /tmp/ncu/c3_full.ncu-rep | tee gpurun_out/r01_c3_gemm_ncu_full.txt
