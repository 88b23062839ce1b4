set -x
mkdir -p gpurun_out
timeout 600 python scripts/p2p_overhead.py 100 20 > gpurun_out/r5a_ovh100.json 2>&1; tail -1 gpurun_out/r5a_ovh100.json
LFOAM_LIB=liblfoam_timing.so timeout 600 python scripts/p2p_overhead.py 100 2 > gpurun_out/r5a_ovh100_timing.log 2>&1; grep -h "LF_TIMING block 0" gpurun_out/r5a_ovh100_timing.log | sed -n '1p;3p;5p;7p'
