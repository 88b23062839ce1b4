set -x
mkdir -p gpurun_out
for lib in liblfoam.so liblfoam_nf.so; do
LFOAM_LIB=$lib timeout 600 python scripts/p2p_overhead.py 200 5 > gpurun_out/r4m_ovh_$lib.json 2>&1; tail -1 gpurun_out/r4m_ovh_$lib.json
done
LFOAM_LIB=liblfoam_timing.so timeout 600 python scripts/p2p_overhead.py 200 2 > gpurun_out/r4m_ovh_timing.log 2>&1; grep -h "LF_TIMING block 0" gpurun_out/r4m_ovh_timing.log | head -20
LFOAM_LIB=liblfoam_nf.so timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_procgeom.py -q -x > gpurun_out/r4m_nf_tests.log 2>&1; tail -2 gpurun_out/r4m_nf_tests.log
