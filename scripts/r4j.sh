set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_procgeom.py -q -rf > gpurun_out/r4j_procgeom.log 2>&1
tail -30 gpurun_out/r4j_procgeom.log
timeout 1500 python -m pytest tests/test_gpu_nonorth.py tests/test_gpu_dtfield.py tests/test_gpu_p2p.py -q -rf > gpurun_out/r4j_regress.log 2>&1
tail -8 gpurun_out/r4j_regress.log
