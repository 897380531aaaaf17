echo "== A: sync after step"; SYNC_AFTER_STEP=1 python tools/dbg_multirank2.py 2>&1 | tail -30
echo "== B: launch blocking test"; CUDA_LAUNCH_BLOCKING=1 python -m pytest tests/test_gpu_multirank.py -q 2>&1 | tail -3
echo "== C: plain"; python tools/dbg_multirank2.py 2>&1 | grep -v "owner 1 pre-gather\|owner 0 pre" | tail -20
