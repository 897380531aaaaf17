ASG_REFRESH=f32 ASG_REFRESH_TIMING=1 timeout 900 python profiles/r01_phase.py step C3 2>&1 | tail -20 | cut -c1-200
