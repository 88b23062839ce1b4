set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 20 --warmup 5 > gpurun_out/r4a_cfg3.json 2> gpurun_out/r4a_cfg3.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r4a_ref3.json 2> gpurun_out/r4a_ref3.err
LFOAM_LIB=liblfoam_timing.so python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/r4a_timing3.log 2>&1
LFOAM_LIB=liblfoam_timing.so python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --config 4 > gpurun_out/r4a_timing4.log 2>&1
python bench.py --steps 10 --warmup 3 --config 4 --no-cpu-baseline > gpurun_out/r4a_cfg4.json 2>&1
tail -c 3000 gpurun_out/r4a_cfg3.json gpurun_out/r4a_ref3.json
grep -h "LF_" gpurun_out/r4a_timing*.log | head -20
