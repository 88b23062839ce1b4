# round-2 check: new tests, full GPU suite, bench configs 3/4/2
timeout 900 python -m pytest tests/test_gpu_hbm.py tests/test_gpu_p2p.py -x -q > gpurun_out/r4b_new.log 2>&1
tail -5 gpurun_out/r4b_new.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r4b_cfg3.json 2> gpurun_out/r4b_cfg3.err
timeout 600 python bench.py --steps 10 --warmup 3 --config 4 --no-cpu-baseline --repeats 2 > gpurun_out/r4b_cfg4.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --config 2 --no-cpu-baseline > gpurun_out/r4b_cfg2.json 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r4b_gpu.log 2>&1
tail -5 gpurun_out/r4b_gpu.log
