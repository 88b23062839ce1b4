#!/bin/bash
# Usage (on the GPU box): scripts/profile_final.sh <tag>
# For every graded workload: the launch list of one bench run (per-launch
# device time + DRAM bytes, cold-cache, serialised) and one `ncu --set full`
# capture of its dominant kernel (+ k_assemble at config 3); summarised ON
# THE BOX into gpurun_out/summary/<tag>_ncu_summary.md and ncu_traffic.json
# (seeded from profiles/, keyed by the device-source hash), keeping only the
# config-3 solve report so gpurun_out stays under the copy-back limit.
set -x
TAG=${1:-final}
OUT=gpurun_out
mkdir -p $OUT/summary
cp profiles/ncu_traffic.json $OUT/summary/ 2>/dev/null
run() {
  local key=$1 kern=$2; shift 2
  local BENCH="python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline $*"
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:'k_(assemble|sum|pcg|gamg|dic)' --csv --log-file $OUT/launches_${TAG}_cfg${key}.csv $BENCH \
     > $OUT/ncu_launch_${TAG}_cfg${key}.log 2>&1
  timeout 1800 ncu --set full --clock-control none --import-source on -k regex:$kern -s 2 -c 1 \
     -o $OUT/prof_${TAG}_cfg${key}_${kern} $BENCH > $OUT/ncu_${TAG}_cfg${key}.log 2>&1
}
run 3 k_pcg_persistent --config 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 3 -c 1 \
   -o $OUT/prof_${TAG}_cfg3_k_assemble python bench.py --steps 3 --warmup 3 --repeats 1 --no-cpu-baseline \
   > $OUT/ncu_${TAG}_cfg3_asm.log 2>&1
run 2 k_pcg_persistent --config 2
run 4 k_pcg_persistent --config 4
run 5 k_pcg_persistent --config 5 --renumber 0
run 5-rcm k_pcg_persistent --config 5 --renumber 1
run 3-dic k_pcg_dic --config 3 --precond DIC
run 4-dic k_pcg_dic --config 4 --precond DIC
run 3-gamg k_pcg_gamg --config 3 --precond GAMG
run 2-corr1 k_pcg_persistent --config 2 --corrected 1
NCU_SUMMARY_DIR=$OUT/summary python scripts/ncu_summary.py $TAG > $OUT/summary/ncu_summary_stdout.log 2>&1
tail -5 $OUT/summary/ncu_summary_stdout.log
for f in $OUT/prof_${TAG}_*.ncu-rep; do
  case $f in *cfg3_k_pcg_persistent*) ;; *) rm -f $f ;; esac
done
du -sh $OUT
