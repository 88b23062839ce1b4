set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_persistent -s 1 -c 1 \
   -o gpurun_out/prof_r4o_p2p200 python scripts/p2p_one.py 200 > gpurun_out/ncu_r4o.log 2>&1
tail -3 gpurun_out/ncu_r4o.log
