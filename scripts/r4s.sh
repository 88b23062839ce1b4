set -x
mkdir -p gpurun_out
BENCH="python bench.py --steps 3 --warmup 3 --repeats 1 --config 3 --no-cpu-baseline"
LFOAM_LIB=liblfoam_uni.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_persistent -s 2 -c 1 \
   -o gpurun_out/prof_r4s_uni $BENCH > gpurun_out/ncu_r4s_uni.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_persistent -s 2 -c 1 \
   -o gpurun_out/prof_r4s_def $BENCH > gpurun_out/ncu_r4s_def.log 2>&1
