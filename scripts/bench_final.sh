#!/bin/bash
# Usage (on the GPU box): scripts/bench_final.sh <tag> — one bench line per graded workload
set -x
TAG=${1:-final}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
b() { local key=$1; shift; timeout 1500 python bench.py "$@" > $OUT/bench_${TAG}_${key}.json 2> $OUT/bench_${TAG}_${key}.err; tail -c 400 $OUT/bench_${TAG}_${key}.json; }
b cfg3
b ref3 --impl reference
b cfg2 --config 2
b cfg4 --config 4 --steps 20 --repeats 2
b cfg5 --config 5 --steps 20 --repeats 2
b cfg5-rcm --config 5 --renumber 1 --steps 20 --repeats 2
b cfg3-dic --config 3 --precond DIC --steps 50 --repeats 3
b cfg4-dic --config 4 --precond DIC --steps 10 --repeats 2
b cfg3-gamg --config 3 --precond GAMG --steps 50 --repeats 3
b cfg2-corr1 --config 2 --corrected 1 --steps 20 --repeats 2
b cfg2-dt --config 2 --dt-field --steps 20 --repeats 2
