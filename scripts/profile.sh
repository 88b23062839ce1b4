#!/bin/bash
# Usage (on the GPU box): scripts/profile.sh <tag> [config]
# 1) launch list with per-launch device time (cold-cache, serialised)
# 2) ncu --set full of the hot kernels (k_phase1, k_phase2, k_assemble)
set -x
TAG=${1:-r1}
CFG=${2:-2}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_(phase|assemble|sum|pcg)' -s 400 -c 300 --csv \
   --log-file $OUT/launches_${TAG}_cfg${CFG}.csv python bench.py --steps 4 --warmup 3 --config $CFG --no-cpu-baseline > $OUT/ncu_launch_${TAG}.log 2>&1
for K in k_phase1 k_phase2 k_assemble; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 2 \
     -o $OUT/prof_${TAG}_cfg${CFG}_${K} python bench.py --steps 2 --warmup 3 --config $CFG --no-cpu-baseline > $OUT/ncu_${K}_${TAG}.log 2>&1
done
ls -la $OUT
