mkdir -p gpurun_out
LFOAM_LIB=liblfoam_timing.so timeout 300 python bench.py --steps 2 --warmup 1 --repeats 1 --no-cpu-baseline > gpurun_out/r6e_c3.log 2>&1
grep -h "LF_TIMING block\|LF_BARRIER" gpurun_out/r6e_c3.log | head -12
LFOAM_LIB=liblfoam_timing.so timeout 300 python bench.py --steps 2 --warmup 1 --repeats 1 --no-cpu-baseline --l2-prefetch 2 > gpurun_out/r6e_c3_nopf.log 2>&1
grep -h "LF_TIMING block\|LF_BARRIER" gpurun_out/r6e_c3_nopf.log | head -12
