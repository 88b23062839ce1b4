#!/bin/bash
# Usage (on the GPU box): scripts/profile_nonorth.sh <tag> [config] [correctors]
# SURVEY §8(f) row 1 workload (skewed graded mesh, corrected laplacian):
# launch list + ncu --set full of the gradient / correction gathers, the
# corrected assembly and the persistent PCG kernel.
set -x
TAG=${1:-r1}
CFG=${2:-2}
NC=${3:-1}
EXTRA=${4:-}          # e.g. --dt-field (then the tag gets -dt)
SUF=""
[ "$EXTRA" = "--dt-field" ] && SUF="-dt"
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 3 --warmup 3 --config $CFG --corrected $NC --no-cpu-baseline $EXTRA"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:'k_(assemble|sum|pcg|grad|lap)' --csv \
   --log-file $OUT/launches_${TAG}_cfg${CFG}-corr${NC}${SUF}.csv $BENCH > $OUT/ncu_launch_${TAG}_cfg${CFG}-corr${NC}${SUF}.log 2>&1
for K in k_grad k_lap_corr k_assemble k_pcg_persistent; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 \
     -o $OUT/prof_${TAG}_cfg${CFG}-corr${NC}${SUF}_${K} $BENCH > $OUT/ncu_${K}_${TAG}_cfg${CFG}-corr${NC}${SUF}.log 2>&1
done
ls -la $OUT
