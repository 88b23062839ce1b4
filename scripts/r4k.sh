set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_p2p.py tests/test_gpu_procgeom.py -q -rf > gpurun_out/r4k_multi.log 2>&1
tail -25 gpurun_out/r4k_multi.log
