# ncu --set full of one wide pair solve and one apply launch of a cold n=2048 solve
mkdir -p gpurun_out /tmp/ncu
ASG_EIGH_DEBUG=1 ASG_EIGH_BATCH=16 ASG_REPS=1 timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  -k regex:"tj_pair_kernel|tj_apply_kernel" -s 20 -c 2 -o /tmp/ncu/tj python profiles/r01_phase.py eigh32 2048 > /tmp/ncu/tj.log 2>&1
tail -2 /tmp/ncu/tj.log
python profiles/ncu_traffic.py /tmp/ncu/tj.ncu-rep > gpurun_out/r01_tj_ncu_full_v9.txt 2>&1
python profiles/ncu_metrics.py /tmp/ncu/tj.ncu-rep "gpu__time_duration.sum$" "bank_conflicts_pipe_lsu_mem_shared.*sum$" \
  "lsu_wavefronts_mem_shared.*sum$" "warp_issue_stalled_.*per_warp_active.pct$" "sm__warps_active.avg.pct_of_peak" \
  "pipe_tensor.*pct_of_peak_sustained_active$" "dram__bytes_(read|write).sum$" "sm__inst_executed.sum$" \
  "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct" "launch__(registers|occupancy_limit)" >> gpurun_out/r01_tj_ncu_full_v9.txt 2>&1
head -60 gpurun_out/r01_tj_ncu_full_v9.txt
