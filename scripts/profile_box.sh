#!/bin/bash
# Usage (on the GPU box): scripts/profile_box.sh <tag> <config...>
# Runs scripts/profile.sh per config, summarises the ncu reports on the box
# (gpurun_out/summary/<tag>_ncu_summary.md, ncu_traffic.json seeded from
# profiles/) and keeps only the k_pcg_persistent reports, so gpurun_out stays
# under the 64 MiB copy-back limit.
TAG=$1; shift
mkdir -p gpurun_out/summary
cp profiles/ncu_traffic.json gpurun_out/summary/ 2>/dev/null
for CFG in "$@"; do
  scripts/profile.sh $TAG $CFG > gpurun_out/${TAG}_prof${CFG}.log 2>&1
done
NCU_SUMMARY_DIR=gpurun_out/summary python scripts/ncu_summary.py $TAG > /dev/null 2>&1
for f in gpurun_out/prof_${TAG}_*.ncu-rep; do
  case $f in *k_pcg_persistent*) ;; *) rm -f $f ;; esac
done
du -sh gpurun_out
