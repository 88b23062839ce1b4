set -x
mkdir -p gpurun_out
timeout 600 python scripts/p2p_overhead.py 200 5 > gpurun_out/r4n_ovh.json 2>&1; tail -1 gpurun_out/r4n_ovh.json
LFOAM_LIB=liblfoam_timing.so timeout 600 python scripts/p2p_overhead.py 200 2 > gpurun_out/r4n_ovh_timing.log 2>&1; grep -h "LF_TIMING block 0" gpurun_out/r4n_ovh_timing.log | sed -n '1p;5p'
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_procgeom.py tests/test_gpu_multi.py tests/test_gpu_dic.py -q -x > gpurun_out/r4n_tests.log 2>&1; tail -2 gpurun_out/r4n_tests.log
