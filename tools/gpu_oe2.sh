# Per-kernel times of the cold tensor-core Jacobi (debug = plain launches, visible to ncu), OE on/off.
mkdir -p gpurun_out
for oe in 0 1; do
  for nb in "512 64" "2048 16"; do
    set -- $nb
    ASG_TJ_OE=$oe ASG_EIGH_DEBUG=1 ASG_EIGH_BATCH=$2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tj_ --csv --log-file /tmp/l_${oe}_$1.csv python profiles/r01_phase.py eigh32 $1 > /dev/null 2>&1
    python profiles/launch_summary.py /tmp/l_${oe}_$1.csv > gpurun_out/oe_${oe}_$1.txt 2>&1; head -6 gpurun_out/oe_${oe}_$1.txt
  done
done
