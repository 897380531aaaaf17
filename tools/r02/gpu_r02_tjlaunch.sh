# Serialised launch list of a warm 2048^2 x 16 eigensolve with the sweeps unrolled (pair vs apply share).
mkdir -p gpurun_out /tmp/ncu
ASG_EIGH_DEBUG=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tj_ -c 20000 --csv --log-file /tmp/ncu/tj.csv \
  python tools/r02/tj_warm.py 2048 16 > /tmp/ncu/tj.log 2>&1
python profiles/launch_summary.py /tmp/ncu/tj.csv > gpurun_out/r02_tj_warm2048_launches_${TAG}.txt 2>&1
head -12 gpurun_out/r02_tj_warm2048_launches_${TAG}.txt
