mkdir -p gpurun_out
LFOAM_LIB=liblfoam_timing.so timeout 300 python bench.py --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline > gpurun_out/r6g_c3.log 2>&1
LFOAM_LIB=liblfoam_timing.so timeout 300 python bench.py --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline --l2-prefetch 2 > gpurun_out/r6g_c3_nopf.log 2>&1
LFOAM_LIB=liblfoam_timing.so timeout 300 python bench.py --config 5 --renumber 1 --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline > gpurun_out/r6g_c5r.log 2>&1
grep -c LF_ARRIVALS gpurun_out/r6g_c3.log
