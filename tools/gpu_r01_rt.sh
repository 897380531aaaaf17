ASG_REFRESH=f32 ASG_REFRESH_TIMING=1 timeout 600 python profiles/r01_phase.py step C2 2>&1 | grep -v "^{" | tail -40
ASG_REFRESH=f32 ASG_REFRESH_TIMING=1 timeout 600 python profiles/r01_phase.py step C1 2>&1 | tail -12
