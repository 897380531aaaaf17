for i in 1 2; do ASG_EIGH_BATCH=64 timeout 900 python profiles/r01_phase.py eigh32 1024 2048 2>&1 | tail -2 | cut -c1-140; done
