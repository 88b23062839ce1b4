#!/bin/bash
# Usage (on the GPU box): scripts/profile.sh <tag> [config]
# 1) launch list with per-launch device time + DRAM bytes (cold-cache, serialised),
#    per-phase launches (--mode graphs) so every kernel kind appears
# 2) ncu --set full of the hot kernels: k_pcg_persistent (default mode),
#    k_phase1 / k_phase2 (graph mode), k_assemble
set -x
TAG=${1:-r1}
CFG=${2:-2}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 3 --warmup 3 --config $CFG --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:'k_(phase|assemble|sum|pcg|amul)' -s 300 -c 400 --csv \
   --log-file $OUT/launches_${TAG}_cfg${CFG}.csv $BENCH --mode graphs > $OUT/ncu_launch_${TAG}_cfg${CFG}.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:'k_(assemble|sum|pcg)' --csv \
   --log-file $OUT/launches_${TAG}_cfg${CFG}_persistent.csv $BENCH > $OUT/ncu_launchp_${TAG}_cfg${CFG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_persistent -s 2 -c 1 \
   -o $OUT/prof_${TAG}_cfg${CFG}_k_pcg_persistent $BENCH > $OUT/ncu_k_pcg_${TAG}_cfg${CFG}.log 2>&1
for K in k_phase1 k_phase2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 50 -c 1 \
     -o $OUT/prof_${TAG}_cfg${CFG}_${K} $BENCH --mode graphs > $OUT/ncu_${K}_${TAG}_cfg${CFG}.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 3 -c 1 \
   -o $OUT/prof_${TAG}_cfg${CFG}_k_assemble $BENCH > $OUT/ncu_k_assemble_${TAG}_cfg${CFG}.log 2>&1
ls -la $OUT
