#!/bin/bash
# Usage (on the GPU box): scripts/profile_dic.sh <tag> [config]
# DIC workload (bench.py --precond DIC, multicolour numbering): launch list
# with per-launch device time + DRAM bytes, and ncu --set full of k_pcg_dic.
set -x
TAG=${1:-r1}
CFG=${2:-2}
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 3 --warmup 3 --config $CFG --precond DIC --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:'k_(assemble|sum|pcg|sym|dic)' --csv \
   --log-file $OUT/launches_${TAG}_cfg${CFG}-dic.csv $BENCH > $OUT/ncu_launch_${TAG}_cfg${CFG}-dic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_dic -s 2 -c 1 \
   -o $OUT/prof_${TAG}_cfg${CFG}-dic_k_pcg_dic $BENCH > $OUT/ncu_k_pcg_dic_${TAG}_cfg${CFG}.log 2>&1
ls -la $OUT
